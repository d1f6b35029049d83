set -u
O=gpurun_out/r2s; mkdir -p $O
for ne in 0 1; do
SGWG_NO_ENERGY=$ne timeout 300 python bench.py --tfinal 1.0 --no-combine --steps 2 --warmup 3 --no-cpu-baseline > $O/bench_ne$ne.json 2> $O/bench_ne$ne.err; echo "rc=$?"
done
