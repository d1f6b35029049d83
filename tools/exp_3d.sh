x() { tail -1 gpurun_out/$1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['ms_per_step'],2), round(d['roofline']['frac'],3))" 2>&1 | tail -1; }
timeout 600 python -m pytest tests/test_gpu_fast.py tests/test_gpu_convergence.py tests/test_gpu_diag.py -q -x > gpurun_out/pytest_3d.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_3d.log
for c in C3 S3; do
timeout 300 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/p3_$c.log 2>&1; x p3_$c.log
SGWG_3D_PIPE=0 timeout 300 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/p3o_$c.log 2>&1; x p3o_$c.log
done
