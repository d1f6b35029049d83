set -u
O=gpurun_out/r2d; mkdir -p $O
for dbg in 0 1 2 3 4 6 7; do
  SGWG_P4_DBG=$dbg timeout 300 python tools/profile_c5.py C5 0.02 > $O/prof_dbg$dbg.json 2>&1; echo "dbg $dbg rc=$?"
done
