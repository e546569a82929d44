set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -40 > gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
timeout 600 python bench.py --steps 30 --warmup 5 --cpu-seconds 10 > gpurun_out/bench.txt 2>&1
tail -5 gpurun_out/pytest_gpu.txt gpurun_out/smoke.txt gpurun_out/bench.txt
