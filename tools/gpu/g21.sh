cd $GRAFT_REPO_ROOT
timeout 600 ncu --set full --import-source on --clock-control none --kernel-name regex:k_fstep16 --launch-skip 6 --launch-count 1 -f -o gpurun_out/r2_fstep16_final python tools/fwd_once.py 4 - 1 > gpurun_out/g21_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --kernel-name regex:k_vmerge --launch-skip 6 --launch-count 1 -f -o gpurun_out/r2_vmerge python tools/fwd_once.py 4 - 1 > gpurun_out/g21_ncu2.log 2>&1
tail -1 gpurun_out/g21_ncu.log
