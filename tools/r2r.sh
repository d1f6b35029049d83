set -u
O=gpurun_out/r2r; mkdir -p $O
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c5_evolve.csv python tools/profile_evolve.py --config C5 --tfinal 0.01 > $O/ncu_le.log 2>&1; echo "ncu launches evolve rc=$?"
timeout 300 python bench.py --tfinal 0.5 --no-combine --steps 2 --warmup 3 --no-cpu-baseline > $O/bench_prefix.json 2> $O/bench_prefix.err; echo "bench prefix rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"field_kernel" -s 3 -c 1 -o $O/field python tools/profile_c5.py C5 0.01 > $O/ncu_field.log 2>&1; echo "ncu field rc=$?"
