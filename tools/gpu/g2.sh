set -x
cd $GRAFT_REPO_ROOT
timeout 300 python tools/ab_solve.py 4 4096 4 "ST_NO_FSTEP16=1" "-" > gpurun_out/g2_ab_small.txt 2>&1
cat gpurun_out/g2_ab_small.txt | tail -5
timeout 300 python tools/ab_solve.py 4 4096 4 "-" "ST_FSTEP_RECOMPUTE=1" >> gpurun_out/g2_ab_small.txt 2>&1
timeout 600 python tools/ab_solve.py 4 32768 32 "ST_NO_FSTEP16=1" "-" > gpurun_out/g2_ab_full.txt 2>&1
timeout 600 python tools/ab_solve.py 4 32768 32 "-" "ST_FSTEP_RECOMPUTE=1" >> gpurun_out/g2_ab_full.txt 2>&1
cat gpurun_out/g2_ab_full.txt | tail -5
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "golden or bf16_configs_reduced or many_blocks or eps_schedule or workspace or reuse" --durations=10 > gpurun_out/g2_pytest.txt 2>&1
tail -25 gpurun_out/g2_pytest.txt
