set -u
O=gpurun_out/r2o; mkdir -p $O
for dbg in 0 8; do
  SGWG_P4_DBG=$dbg timeout 300 python tools/profile_c5.py C5 0.02 > $O/prof_d$dbg.json 2>&1; echo "d $dbg rc=$?"
done
SGWG_P4_XTARGET=3072 timeout 300 python tools/profile_c5.py C5 0.02 > $O/prof_xt3072.json 2>&1; echo "rc=$?"
