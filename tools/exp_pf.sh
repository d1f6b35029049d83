x() { tail -1 gpurun_out/$1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['ms_per_step'],2), round(d['roofline']['frac'],3))"; }
timeout 600 python -m pytest tests/test_gpu_vp.py tests/test_gpu_landau.py -q -x > gpurun_out/pytest_vp.log 2>&1; tail -2 gpurun_out/pytest_vp.log
B="python bench.py --config C5 --tfinal 0.05 --no-combine --steps 3 --warmup 3 --no-cpu-baseline"
timeout 300 $B > gpurun_out/p_base.log 2>&1; x p_base.log
SGWG_LIB=paper_2007_10196_b200/libsgwg_pf.so timeout 300 $B > gpurun_out/p_pf.log 2>&1; x p_pf.log
timeout 300 $B > gpurun_out/p_base2.log 2>&1; x p_base2.log
SGWG_LIB=paper_2007_10196_b200/libsgwg_pf.so timeout 300 $B > gpurun_out/p_pf2.log 2>&1; x p_pf2.log
