cd $GRAFT_REPO_ROOT
timeout 300 python tools/ab_solve.py 4 32768 32 "ST_NO_FSTEP16=1" "-" > gpurun_out/g8_ab.txt 2>&1
tail -1 gpurun_out/g8_ab.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "golden or bf16_configs_reduced or many_blocks or eps_schedule or workspace or reuse" > gpurun_out/g8_pytest.txt 2>&1
tail -3 gpurun_out/g8_pytest.txt
timeout 600 ncu --set full --import-source on --clock-control none --kernel-name regex:k_fstep16 --launch-skip 6 --launch-count 1 -f -o gpurun_out/r2_fstep16f python tools/fwd_once.py 4 - 1 > gpurun_out/g8_ncu.log 2>&1
tail -2 gpurun_out/g8_ncu.log
