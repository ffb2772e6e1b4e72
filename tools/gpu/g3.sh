cd $GRAFT_REPO_ROOT
for d in 0 1 2 4 5 3; do
  echo "dbg=$d" >> gpurun_out/g3_abl.txt
  ST_PHASE_DBG=$d timeout 300 python tools/ab_solve.py 4 32768 32 "-" "-" 2>&1 | tail -1 >> gpurun_out/g3_abl.txt
done
cat gpurun_out/g3_abl.txt
timeout 600 ncu --set full --import-source on --kernel-name regex:k_fstep16 --launch-skip 6 --launch-count 1 -f -o gpurun_out/r2_fstep16 python tools/fwd_once.py 4 - 1 > gpurun_out/g3_ncu.log 2>&1
tail -3 gpurun_out/g3_ncu.log
