set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/g1_pytest.txt
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/g1_bench4.json 2> gpurun_out/g1_bench4.err
tail -c 3000 gpurun_out/g1_bench4.err
cat gpurun_out/g1_bench4.json | head -c 4000
