set -u
mkdir -p gpurun_out/g1
nvidia-smi --query-gpu=name,clocks.sm,memory.total --format=csv > gpurun_out/g1/smi.txt 2>&1
timeout 600 python tools/c5_combine.py fast > gpurun_out/g1/c5_combine.log 2>&1; echo "c5comb rc=$?"
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/g1/pytest.log 2>&1; echo "pytest rc=$?"
