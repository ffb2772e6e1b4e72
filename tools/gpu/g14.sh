cd $GRAFT_REPO_ROOT
export ST_PARITY_OUT=gpurun_out/r2_parity.json
timeout 1800 python -m pytest tests -m gpu -x -q --durations=15 -k "not sanitizer" > gpurun_out/g14_pytest.txt 2>&1
tail -25 gpurun_out/g14_pytest.txt
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/g14_bench.json 2> gpurun_out/g14_bench.err
tail -c 1500 gpurun_out/g14_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_launches_config4.csv python tools/fwd_once.py 4 - 1 > gpurun_out/g14_ncu.log 2>&1
tail -2 gpurun_out/g14_ncu.log
