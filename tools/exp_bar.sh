x() { tail -1 gpurun_out/$1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['ms_per_step'],2), round(d['roofline']['frac'],3))"; }
timeout 600 python -m pytest tests/test_gpu_fast.py tests/test_gpu_parity.py -q -x > gpurun_out/pytest_bar.log 2>&1; tail -2 gpurun_out/pytest_bar.log
for c in C2 C1; do
timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b_new_$c.log 2>&1; x b_new_$c.log
SGWG_LIB=paper_2007_10196_b200/libsgwg_cg.so timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b_cg_$c.log 2>&1; x b_cg_$c.log
done
SGWG_LIB=paper_2007_10196_b200/libsgwg_tr.so timeout 300 python tools/trace_c2.py C2
