cd $GRAFT_REPO_ROOT
ST_TRACE_FSTEP=50 timeout 300 python tools/time_fwd.py 4 2>&1 | head -12 > gpurun_out/g12.txt
