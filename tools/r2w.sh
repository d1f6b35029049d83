set -u
O=gpurun_out/r2w; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_vp.py tests/test_gpu_landau.py tests/test_gpu_multirank.py -q -x > $O/tests.log 2>&1; echo "tests rc=$?"
for ov in 0 1; do
SGWG_P4_OVERLAP=$ov timeout 300 python bench.py --tfinal 1.0 --no-combine --steps 2 --warmup 3 --no-cpu-baseline > $O/bench_ov$ov.json 2> $O/bench_ov$ov.err; echo "rc=$?"
done
