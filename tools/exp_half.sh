# 1024-point (two CTAs/SM) vs 2048-point 2D stage tiles on the large / non-persistent 2D cases
x() { tail -1 gpurun_out/$1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; s=r.get('single_stage_launch',{}); print('$1', round(d['ms_per_step'],2), round(r['frac'],3), 'stage', round(s.get('avg_launch_us',0),1), round(s.get('frac',0),3))"; }
mkdir -p gpurun_out/half
timeout 900 python -m pytest tests/test_gpu_fast.py tests/test_gpu_vp.py -q -x > gpurun_out/half/pytest.log 2>&1; tail -1 gpurun_out/half/pytest.log
for c in S2 C4; do
  SGWG_TILE2D=2048 timeout 300 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/half/${c}_2048.log 2>&1; x half/${c}_2048.log
  timeout 300 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/half/${c}_1024.log 2>&1; x half/${c}_1024.log
done
SGWG_NO_PERSIST=1 timeout 300 python bench.py --config C2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/half/C2np_1024.log 2>&1; x half/C2np_1024.log
SGWG_NO_PERSIST=1 SGWG_TILE2D=2048 timeout 300 python bench.py --config C2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/half/C2np_2048.log 2>&1; x half/C2np_2048.log
