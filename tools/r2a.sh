set -u
O=gpurun_out/r2a; mkdir -p $O
nproc > $O/nproc.txt; nvidia-smi > $O/smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 300 python tools/profile_c5.py C5 0.02 > $O/prof.json 2> $O/prof.err; echo "prof rc=$?"
( time timeout 1200 python bench.py > $O/bench.json 2> $O/bench.err ) 2> $O/bench.time; echo "bench rc=$?"
timeout 1800 python -m pytest tests -m gpu -q -s --durations=30 > $O/pytest.log 2>&1; echo "pytest rc=$?"
