set -u
mkdir -p gpurun_out/g2
nproc > gpurun_out/g2/nproc.txt
timeout 1500 python -m pytest tests/test_gpu_fullsize_parity.py -q -s > gpurun_out/g2/full.log 2>&1; echo "full rc=$?"
