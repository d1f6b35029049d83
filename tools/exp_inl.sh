x() { tail -1 gpurun_out/$1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['ms_per_step'],2), round(d['roofline']['frac'],3))"; }
timeout 900 python -m pytest tests/test_gpu_convergence.py -q -x > gpurun_out/pytest_conv.log 2>&1; tail -2 gpurun_out/pytest_conv.log
for c in C5 C2 C3; do
  extra=""; [ $c = C5 ] && extra="--tfinal 0.05 --no-combine"
  timeout 300 python bench.py --config $c $extra --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/i_base_$c.log 2>&1; x i_base_$c.log
  SGWG_LIB=paper_2007_10196_b200/libsgwg_inl.so timeout 300 python bench.py --config $c $extra --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/i_inl_$c.log 2>&1; x i_inl_$c.log
done
