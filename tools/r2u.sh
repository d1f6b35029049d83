set -u
O=gpurun_out/r2u; mkdir -p $O
for c in C1 C2 C3 C4 S2 S3; do
  timeout 900 python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.err; echo "$c rc=$?"
done
timeout 900 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err; echo "ref rc=$?"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_bench_default.csv python bench.py --tfinal 0.02 --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline > $O/ncu_bench.log 2>&1; echo "ncu bench rc=$?"
