cd $GRAFT_REPO_ROOT
python tools/time_fwd.py 4 > gpurun_out/g13.txt 2>&1
timeout 600 ncu --set full --import-source on --clock-control none --kernel-name regex:k_fstep16 --launch-skip 6 --launch-count 1 -f -o gpurun_out/r2_fstep16g python tools/fwd_once.py 4 - 1 > gpurun_out/g13_ncu.log 2>&1
tail -1 gpurun_out/g13_ncu.log
