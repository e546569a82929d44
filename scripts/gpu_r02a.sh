# r02 first check: full GPU tests, smoke, quick bench, workloads
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -q -rf > $OUT/pytest_gpu.txt 2>&1; tail -15 $OUT/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py > $OUT/bench_default.txt 2>&1; tail -1 $OUT/bench_default.txt
