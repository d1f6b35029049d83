set -u
O=gpurun_out/r2k; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?"
timeout 300 python tools/profile_c5.py C5 0.02 > $O/prof.json 2>&1; echo "prof rc=$?"
( time timeout 1200 python bench.py > $O/bench.json 2> $O/bench.err ) 2> $O/bench.time; echo "bench rc=$?"
