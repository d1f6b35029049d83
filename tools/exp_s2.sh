x() { tail -1 gpurun_out/$1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['ms_per_step'],2), round(d['roofline']['frac'],3), d['roofline'].get('kernel','')[:40])"; }
timeout 600 python -m pytest tests/test_gpu_fast.py -q -x > gpurun_out/pytest_fast.log 2>&1; tail -1 gpurun_out/pytest_fast.log
for c in S2 C2 C1; do timeout 300 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/s2_$c.log 2>&1; x s2_$c.log; done
