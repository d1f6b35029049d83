B="python bench.py --config C4 --steps 2 --warmup 3 --no-cpu-baseline"
x() { tail -1 gpurun_out/$1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['ms_per_step'],2))"; }
SGWG_LIB=paper_2007_10196_b200/libsgwg_old.so timeout 200 $B > gpurun_out/c4_old.log 2>&1; x c4_old.log
timeout 200 $B > gpurun_out/c4_new.log 2>&1; x c4_new.log
SGWG_LIB=paper_2007_10196_b200/libsgwg_old.so timeout 200 $B > gpurun_out/c4_old2.log 2>&1; x c4_old2.log
SGWG_LIB=paper_2007_10196_b200/libsgwg_old.so timeout 200 python bench.py --config C2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/c2_old.log 2>&1; x c2_old.log
timeout 200 python bench.py --config C2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/c2_new.log 2>&1; x c2_new.log
