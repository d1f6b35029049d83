set -u
O=gpurun_out/r2t; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_landau.py tests/test_gpu_vp.py -q -x > $O/tests.log 2>&1; echo "tests rc=$?"
for ne in 0 1; do
SGWG_NO_ENERGY=$ne timeout 300 python bench.py --tfinal 1.0 --no-combine --steps 2 --warmup 3 --no-cpu-baseline > $O/bench_ne$ne.json 2> $O/bench_ne$ne.err; echo "rc=$?"
done
