x() { tail -1 gpurun_out/$1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['ms_per_step'],2), d.get('gpu_launches'))" 2>&1 | tail -1; }
B="python bench.py --config C4 --steps 2 --warmup 3 --no-cpu-baseline"
timeout 300 $B > gpurun_out/c4_tail.log 2>&1; x c4_tail.log
SGWG_VP_FIELD_TAIL=0 timeout 300 $B > gpurun_out/c4_notail.log 2>&1; x c4_notail.log
SGWG_VP_FUSE_MOMENT=1 timeout 300 $B > gpurun_out/c4_fm.log 2>&1; x c4_fm.log
