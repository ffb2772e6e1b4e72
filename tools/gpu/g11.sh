cd $GRAFT_REPO_ROOT
timeout 300 python tools/time_fwd.py 4 > gpurun_out/g11.txt 2>&1
ST_TRACE_FSTEP=50 timeout 300 python tools/time_fwd.py 4 2>&1 | head -12 >> gpurun_out/g11.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "golden or bf16_configs_reduced or many_blocks or eps_schedule or workspace or reuse" > gpurun_out/g11_pytest.txt 2>&1
tail -3 gpurun_out/g11_pytest.txt
cat gpurun_out/g11.txt
