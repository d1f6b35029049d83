x() { tail -1 gpurun_out/$1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['ms_per_step'],2))" 2>&1 | tail -1; }
B="python bench.py --config C4 --steps 2 --warmup 3 --no-cpu-baseline"
timeout 300 $B > gpurun_out/c4e.log 2>&1; x c4e.log
SGWG_CARVEOUT=1 timeout 300 $B > gpurun_out/c4f.log 2>&1; x c4f.log
SGWG_CARVEOUT=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4d.csv python bench.py --config C4 --tfinal 0.05 --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_c4.log 2>&1
