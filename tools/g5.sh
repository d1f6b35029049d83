set -u
O=gpurun_out/g5; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_vp.py -q -x > $O/vp.log 2>&1; echo "vp rc=$?"
timeout 300 python tools/profile_c5.py C5 0.02 > $O/prof.json 2> $O/prof.err; echo "prof rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"xpass4d|vpass4d" -s 6 -c 2 -o $O/p4 python tools/profile_c5.py C5 0.01 > $O/ncu.log 2>&1; echo "ncu rc=$?"
timeout 900 python bench.py --tfinal 0.2 --steps 2 --warmup 3 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
