# Round-end measurement set (one GPU): the default bench line, the reference
# arm, every config's bench line, the launch list of the default bench command
# and one full ncu capture of its dominant kernel.
set -u
O=gpurun_out/final
mkdir -p $O
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "default rc=$?"
timeout 900 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err; echo "reference rc=$?"
for c in C1 C3 C4 S2 S3; do
  timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; echo "$c rc=$?"
done
timeout 600 python bench.py --config C5 --tfinal 0.05 --no-combine --steps 3 --warmup 3 > $O/bench_C5.json 2> $O/bench_C5.err; echo "C5 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_bench_default.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline > $O/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:evolve2d_persistent -c 1 -o $O/prof_persist_c2 python bench.py --steps 1 --warmup 0 --no-cpu-baseline > $O/ncu_full.log 2>&1; echo "ncu full rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:plane_fast -c 2 -o $O/prof_plane_c5 python tools/profile_case.py --config C5 --steps 1 --no-combine > $O/ncu_plane.log 2>&1; echo "ncu plane rc=$?"
