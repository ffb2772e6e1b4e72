# Round-2 evidence on one B200 (run under gpurun from the repo root): timings, bench (both arms), the ncu
# launch list of the bench command, backward launch lists, ncu --set full summaries of the dominant kernels.
set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out /tmp/ncu
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "reuse or band_free" > gpurun_out/quick_tests.log 2>&1; tail -2 gpurun_out/quick_tests.log
python tools/timing.py 1 2 3 4 5 > gpurun_out/r2_configs_timing.txt 2>&1
BWD_MODE=direct_four_plan python tools/timing.py 2 4 5 >> gpurun_out/r2_configs_timing.txt 2>&1
python bench.py > gpurun_out/r2_bench_config4.json 2> gpurun_out/bench.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2_bench_reference.json 2> gpurun_out/bench_ref.err
python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_step_config4.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_launch.log 2>&1
python tools/launch_table.py gpurun_out/r2_launches_step_config4.csv > gpurun_out/r2_launches_step_config4.txt
for c in 4 5; do
  python tools/bwd_only.py $c > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bwd_c$c.csv python tools/bwd_only.py $c > /dev/null 2>&1
  python tools/launch_table.py gpurun_out/bwd_c$c.csv > gpurun_out/r2_launches_bwd_config$c.txt
done
python tools/bwd_only.py 4 direct_four_plan > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bwd_c4d.csv python tools/bwd_only.py 4 direct_four_plan > /dev/null 2>&1
python tools/launch_table.py gpurun_out/bwd_c4d.csv > gpurun_out/r2_launches_bwd_config4_direct.txt
bash tools/gpu/r2_ncu_bsweep.sh > gpurun_out/ncu_bsweep_all.log 2>&1
timeout 600 ncu --set full --clock-control none --kernel-name regex:k_fstep16 --launch-skip 4 --launch-count 1 -f -o /tmp/ncu/fstep python tools/fwd_short.py 4 > gpurun_out/ncu_fstep.log 2>&1
python tools/ncu_summary.py /tmp/ncu/fstep.ncu-rep > gpurun_out/r2_ncu_config4_fstep16.txt 2>&1
cat gpurun_out/r2_configs_timing.txt
