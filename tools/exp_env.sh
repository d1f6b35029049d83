# env A/B on one build: bash tools/exp_env.sh "ENV=1 ..." "pytest files" CFG...
x() { tail -1 gpurun_out/$1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$1', round(d['ms_per_step'],3), 'frac', round(r['frac'],3))"; }
mkdir -p gpurun_out/env
E="$1"; T="$2"; shift 2
if [ -n "$T" ]; then env $E timeout 1200 python -m pytest $T -q -x > gpurun_out/env/pytest.log 2>&1; tail -1 gpurun_out/env/pytest.log; fi
for c in "$@"; do
  a="--steps 5 --warmup 3 --no-cpu-baseline"
  timeout 600 python bench.py --config $c $a > gpurun_out/env/${c}_base.log 2>&1; x env/${c}_base.log
  env $E timeout 600 python bench.py --config $c $a > gpurun_out/env/${c}_env.log 2>&1; x env/${c}_env.log
  timeout 600 python bench.py --config $c $a > gpurun_out/env/${c}_base2.log 2>&1; x env/${c}_base2.log
done
