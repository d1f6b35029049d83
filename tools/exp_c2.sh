x() { tail -1 gpurun_out/$1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['ms_per_step'],2), round(d['roofline']['frac'],3))" 2>&1 | tail -1; }
timeout 600 python -m pytest tests/test_gpu_fast.py -q -x > gpurun_out/pytest_c2.log 2>&1; echo "pytest rc=$?"
for i in 1 2; do timeout 200 python bench.py --config C2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/c2_$i.log 2>&1; x c2_$i.log; done
timeout 200 python bench.py --config S2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/s2x.log 2>&1; x s2x.log
