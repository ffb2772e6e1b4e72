cd $GRAFT_REPO_ROOT
ST_TRACE_FSTEP=50 timeout 300 python tools/time_fwd.py 4 > gpurun_out/g10.txt 2>&1
cat gpurun_out/g10.txt | head -60
