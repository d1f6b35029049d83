# library A/B: bash tools/exp_lib.sh <variant.so> CFG... (base = libsgwg.so)
x() { tail -1 gpurun_out/$1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['ms_per_step'],3))" 2>/dev/null || echo "$1 FAILED"; }
mkdir -p gpurun_out/lib
V="$1"; shift
for c in "$@"; do
  a="--config $c --steps 3 --warmup 3 --no-cpu-baseline"
  [ "$c" = "C5" ] && a="$a --tfinal 0.05 --no-combine"
  timeout 600 python bench.py $a > gpurun_out/lib/${c}_base.log 2>&1; x lib/${c}_base.log
  SGWG_LIB=$V timeout 600 python bench.py $a > gpurun_out/lib/${c}_var.log 2>&1; x lib/${c}_var.log
  timeout 600 python bench.py $a > gpurun_out/lib/${c}_base2.log 2>&1; x lib/${c}_base2.log
done
