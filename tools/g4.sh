set -u
O=gpurun_out/g4; mkdir -p $O
timeout 300 python tools/profile_c5.py C5 0.02 > $O/prof.json 2> $O/prof.err; echo "prof rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"xpass4d|vpass4d" -s 6 -c 2 -o $O/p4 python tools/profile_c5.py C5 0.01 > $O/ncu.log 2>&1; echo "ncu rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python tools/profile_evolve.py --config C5 --tfinal 0.01 > $O/ncu_l.log 2>&1; echo "ncu launches rc=$?"
