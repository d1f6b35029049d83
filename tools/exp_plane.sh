# plane-kernel CTA size variants on C5 (prefix T=0.05, no combine)
x() { tail -1 gpurun_out/$1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['ms_per_step'],3))" 2>/dev/null || echo "$1 FAILED"; }
mkdir -p gpurun_out/plane
A="--config C5 --tfinal 0.05 --no-combine --steps 3 --warmup 3 --no-cpu-baseline"
timeout 300 python bench.py $A > gpurun_out/plane/base.log 2>&1; x plane/base.log
SGWG_LIB=paper_2007_10196_b200/libsgwg_p128.so SGWG_PLANE_CAP=1024 SGWG_PLANE_SMEM=4500 timeout 300 python bench.py $A > gpurun_out/plane/p128.log 2>&1; x plane/p128.log
SGWG_LIB=paper_2007_10196_b200/libsgwg_p128b.so SGWG_PLANE_CAP=1024 SGWG_PLANE_SMEM=5400 timeout 300 python bench.py $A > gpurun_out/plane/p128b.log 2>&1; x plane/p128b.log
SGWG_LIB=paper_2007_10196_b200/libsgwg_p128.so SGWG_PLANE_CAP=1024 SGWG_PLANE_SMEM=4500 timeout 600 python -m pytest tests/test_gpu_vp.py -q -x -k c5 2>&1 | tail -1
timeout 300 python bench.py $A > gpurun_out/plane/base2.log 2>&1; x plane/base2.log
