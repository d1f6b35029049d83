set -u
O=gpurun_out/r2y; mkdir -p $O
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"xpass4d_kernel|vpass4d_persist|field_kernel|energy_rows" -s 8 -c 4 -o $O/c5 python tools/profile_evolve.py --config C5 --tfinal 0.01 > $O/ncu_c5.log 2>&1; echo "ncu c5 rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"final_fast|upsample_fast" -c 4 -o $O/comb python tools/c5_combine.py fast > $O/ncu_comb.log 2>&1; echo "ncu comb rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"stage3d_small|evolve2d_persistent" -s 3 -c 1 -o $O/c3 python tools/profile_evolve.py --config C3 --tfinal 0.005 > $O/ncu_c3.log 2>&1; echo "ncu c3 rc=$?"
