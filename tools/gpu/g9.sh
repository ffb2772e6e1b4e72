cd $GRAFT_REPO_ROOT
for d in 0 1 2 3; do ST_PHASE_DBG=$d timeout 300 python tools/time_fwd.py 4 >> gpurun_out/g9.txt 2>&1; done
cat gpurun_out/g9.txt
