set -u
O=gpurun_out/r2b; mkdir -p $O
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c5_evolve.csv python tools/profile_evolve.py --config C5 --tfinal 0.01 > $O/ncu_le.log 2>&1; echo "ncu launches evolve rc=$?"
timeout 600 python tools/c5_combine.py fast > $O/c5_combine.log 2>&1; echo "c5comb rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c5_combine.csv python tools/c5_combine.py fast > $O/ncu_lc.log 2>&1; echo "ncu launches comb rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"xpass4d|vpass4d" -s 6 -c 2 -o $O/p4 python tools/profile_c5.py C5 0.01 > $O/ncu_p4.log 2>&1; echo "ncu p4 rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"upsample|final_fast" -c 4 -o $O/comb python tools/c5_combine.py fast > $O/ncu_comb.log 2>&1; echo "ncu comb rc=$?"
