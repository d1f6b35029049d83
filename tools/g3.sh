set -u
O=gpurun_out/r3j; mkdir -p $O
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"xpass4d_kernel|vpass4d_persist" -s 8 -c 2 -o $O/c5 python tools/profile_evolve.py --config C5 --tfinal 0.01 > $O/ncu_c5.log 2>&1; echo "ncu c5 rc=$?"
ls -la $O
