set -u
O=gpurun_out/r2c; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_vp.py tests/test_gpu_hardening.py -q -x > $O/tests.log 2>&1; echo "tests rc=$?"
for rpt in 1 2 4; do
  SGWG_P4_RPT=$rpt timeout 300 python tools/profile_c5.py C5 0.02 > $O/prof_rpt$rpt.json 2>&1; echo "rpt $rpt rc=$?"
done
for vt in 1800 3000; do
  SGWG_P4_VTARGET=$vt timeout 300 python tools/profile_c5.py C5 0.02 > $O/prof_vt$vt.json 2>&1; echo "vt $vt rc=$?"
done
for xt in 2048 8192; do
  SGWG_P4_XTARGET=$xt timeout 300 python tools/profile_c5.py C5 0.02 > $O/prof_xt$xt.json 2>&1; echo "xt $xt rc=$?"
done
