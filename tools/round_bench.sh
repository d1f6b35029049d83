# Round-end measurement set (one GPU): the GPU test suite, the default bench line (C5), the
# reference arm, every other config's bench line, the launch lists of a C5 evolve and of the
# C5 combination, and full ncu captures of the C5 kernels.  Output: gpurun_out/final/.
set -u
O=gpurun_out/final
mkdir -p $O
timeout 2400 python -m pytest tests -x -q -m gpu > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_gpu.log
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "default rc=$?"
timeout 900 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err; echo "reference rc=$?"
for c in C1 C2 C3 C4 S2 S3; do
  timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; echo "$c rc=$?"
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c5_evolve.csv python tools/profile_evolve.py --config C5 --tfinal 0.012 > $O/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"xpass4d_kernel|vpass4d_persist|field_kernel|energy_rows_batch|group_batch" -s 8 -c 6 -o $O/c5 python tools/profile_evolve.py --config C5 --tfinal 0.15 > $O/ncu_c5.log 2>&1; echo "ncu c5 rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"final_fast|upsample_fast" -c 4 -o $O/comb python tools/c5_combine.py fast > $O/ncu_comb.log 2>&1; echo "ncu comb rc=$?"
