# ncu --set full of the band-free sweeps (config 4): launch order of k_bsweep in tools/bwd_only.py is
# RO | C1 R12 C3 R4 R6 C6 | C1 R12 C3 R4 R6 C6  -> skip 7 = C1 (PV), 8 = R12, 9 = C3 (PX), 11 = R6 (SBAR row)
set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out /tmp/ncu
for pair in "7 pv_c1" "8 r12" "9 px_c3" "11 sbar_r6"; do
  set -- $pair
  timeout 600 ncu --set full --clock-control none --import-source on --kernel-name regex:k_bsweep --launch-skip $1 --launch-count 1 -f -o /tmp/ncu/$2 python tools/bwd_only.py 4 > gpurun_out/ncu_$2.log 2>&1
  python tools/ncu_summary.py /tmp/ncu/$2.ncu-rep > gpurun_out/r2_ncu_config4_bsweep_$2.txt 2>&1
done

cat gpurun_out/r2_ncu_config4_bsweep_*.txt
