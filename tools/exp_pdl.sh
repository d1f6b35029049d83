x() { tail -1 gpurun_out/$1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['ms_per_step'],2))" 2>&1 | tail -1; }
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_pdl.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_pdl.log
for c in C4 C3 C5; do
  extra=""; [ $c = C5 ] && extra="--tfinal 0.05 --no-combine"
  timeout 300 python bench.py --config $c $extra --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/pdl_$c.log 2>&1; x pdl_$c.log
  SGWG_PDL=0 timeout 300 python bench.py --config $c $extra --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/nopdl_$c.log 2>&1; x nopdl_$c.log
done
