set -u
O=gpurun_out/g3; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_vp.py tests/test_gpu_fullsize.py -q -x > $O/vp.log 2>&1; echo "vp rc=$?"
for p4 in 1 0; do
SGWG_PLANE4=$p4 timeout 300 python bench.py --config C5 --tfinal 0.05 --no-combine --steps 3 --warmup 3 --no-cpu-baseline > $O/c5_p4_$p4.json 2> $O/c5_p4_$p4.err; echo "c5 p4=$p4 rc=$?"
done
timeout 900 python -m pytest tests/test_gpu_fullsize_parity.py -q -s -k c5 > $O/full_c5.log 2>&1; echo "fullc5 rc=$?"
