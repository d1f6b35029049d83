# A/B: libsgwg_old.so (last commit) vs the working tree's libsgwg.so on the given configs
# usage: bash tools/exp_ab.sh "pytest files" CFG...
x() { tail -1 gpurun_out/$1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; s=r.get('single_stage_launch',{}); print('$1', round(d['ms_per_step'],3), 'frac', round(r['frac'],3), 'stage_us', round(s.get('avg_launch_us',0),1), round(s.get('frac',0),3))"; }
mkdir -p gpurun_out/ab
T="$1"; shift
if [ -n "$T" ]; then timeout 1200 python -m pytest $T -q -x > gpurun_out/ab/pytest.log 2>&1; tail -1 gpurun_out/ab/pytest.log; fi
for c in "$@"; do
  a="--steps 3 --warmup 3 --no-cpu-baseline"
  [ "$c" = "C5" ] && a="$a --tfinal 0.05 --no-combine"
  SGWG_LIB=paper_2007_10196_b200/libsgwg_old.so timeout 600 python bench.py --config $c $a > gpurun_out/ab/${c}_old.log 2>&1; x ab/${c}_old.log
  timeout 600 python bench.py --config $c $a > gpurun_out/ab/${c}_new.log 2>&1; x ab/${c}_new.log
done
