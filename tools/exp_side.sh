x() { tail -1 gpurun_out/$1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['ms_per_step'],2))" 2>&1 | tail -1; }
timeout 900 python -m pytest tests/test_gpu_landau.py tests/test_gpu_vp.py tests/test_gpu_runner.py tests/test_gpu_fullsize.py -q -x > gpurun_out/pytest_side.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_side.log
timeout 300 python bench.py --config C4 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/side_C4.log 2>&1; x side_C4.log
timeout 300 python bench.py --config C5 --tfinal 0.05 --no-combine --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/side_C5.log 2>&1; x side_C5.log
