set -u
O=gpurun_out/r2i; mkdir -p $O
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"vpass4d" -s 3 -c 1 -o $O/vp python tools/profile_c5.py C5 0.01 > $O/ncu_vp.log 2>&1; echo "ncu rc=$?"
