set -u
O=gpurun_out/r3q; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_landau.py tests/test_gpu_vp.py -x -q -m gpu > $O/pytest_l.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_l.log
timeout 900 python -m pytest tests/test_gpu_fullsize_parity.py -x -q -m gpu -k "c4" > $O/pytest_c4.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_c4.log
for b in 1 0; do
SGWG_ENERGY_BATCH=$b timeout 600 python bench.py --config C4 --steps 2 --warmup 3 --no-cpu-baseline > $O/bench_C4_b$b.json 2> $O/bench_C4_b$b.err; echo "C4 batch=$b rc=$?"; python -c "
import json;d=json.load(open('$O/bench_C4_b$b.json'));print(d['ms_per_step'],d['value'],d['gpu_launches'])"
done
