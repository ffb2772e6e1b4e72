cd $GRAFT_REPO_ROOT
for c in 4 5 2; do
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv --log-file gpurun_out/r2_launches_step_config$c.csv python tools/bwd_once.py $c > gpurun_out/g19_ncu$c.log 2>&1
done
python tools/timing.py 1 2 3 4 5 > gpurun_out/r2_timing.txt 2>&1; BWD_MODE=direct_four_plan python tools/timing.py 4 5 >> gpurun_out/r2_timing.txt 2>&1
tail -3 gpurun_out/g19_ncu4.log
