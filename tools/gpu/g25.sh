cd $GRAFT_REPO_ROOT
mkdir -p /tmp/ncu
timeout 900 ncu --set full --clock-control none --kernel-name regex:k_bwdM --launch-count 1 -f -o /tmp/ncu/bwdM python tools/bwd_once.py 4 > gpurun_out/g25.log 2>&1
timeout 900 ncu --set full --clock-control none --kernel-name regex:k_sweepW --launch-count 1 -f -o /tmp/ncu/sweepW python tools/bwd_once.py 4 >> gpurun_out/g25.log 2>&1
python tools/ncu_summary.py /tmp/ncu/bwdM.ncu-rep > gpurun_out/r2_ncu_config4_bwdM.txt 2>&1
python tools/ncu_summary.py /tmp/ncu/sweepW.ncu-rep > gpurun_out/r2_ncu_config4_sweepW.txt 2>&1
ncu -i /tmp/ncu/bwdM.ncu-rep --page details --csv > gpurun_out/r2_bwdM_details.csv 2>&1
