set -u
O=gpurun_out/r2m; mkdir -p $O
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"final_fast|upsample_fast" -c 4 -o $O/comb python tools/c5_combine.py fast > $O/ncu_comb.log 2>&1; echo "ncu comb rc=$?"
