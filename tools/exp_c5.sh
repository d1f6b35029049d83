set -x
B="python bench.py --config C5 --tfinal 0.05 --no-combine --steps 3 --warmup 3 --no-cpu-baseline"
x() { tail -1 gpurun_out/$1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['ms_per_step'],2))"; }
timeout 600 python -m pytest tests/test_gpu_landau.py tests/test_gpu_vp.py -q -x > gpurun_out/pytest_field.log 2>&1; tail -2 gpurun_out/pytest_field.log
timeout 200 $B > gpurun_out/e_base.log 2>&1; x e_base.log
SGWG_PLANE_CAP=1024 timeout 200 $B > gpurun_out/e_c1024.log 2>&1; x e_c1024.log
SGWG_LIB=paper_2007_10196_b200/libsgwg_v4.so SGWG_PLANE_SMEM=7000 timeout 200 $B > gpurun_out/e_v4.log 2>&1; x e_v4.log
SGWG_LIB=paper_2007_10196_b200/libsgwg_v4.so SGWG_PLANE_SMEM=7000 SGWG_PLANE_CAP=1024 timeout 200 $B > gpurun_out/e_v4c.log 2>&1; x e_v4c.log
timeout 300 python bench.py --config C4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4.log 2>&1; x bench_c4.log
