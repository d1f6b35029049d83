x() { tail -1 gpurun_out/$1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['ms_per_step'],2), round(d['roofline']['frac'],3))" 2>&1 | tail -1; }
timeout 300 python -m pytest tests/test_gpu_fast.py -q -x > gpurun_out/pytest_ms.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_ms.log
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "stop or persist or fast" > gpurun_out/pytest_ms2.log 2>&1; echo "pytest2 rc=$?"; tail -2 gpurun_out/pytest_ms2.log
for c in C2 C1; do
timeout 200 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ms_on_$c.log 2>&1; x ms_on_$c.log
SGWG_MEMBER_SYNC=0 timeout 200 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ms_off_$c.log 2>&1; x ms_off_$c.log
done
