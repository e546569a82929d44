# Round-end style check: GPU tests, smoke, default bench (with CPU baseline),
# reference arm.
OUT=gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.txt 2>&1; tail -2 $OUT/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > $OUT/bench_default.txt 2>&1; tail -1 $OUT/bench_default.txt
timeout 600 python bench.py --impl reference > $OUT/bench_reference.txt 2>&1; tail -1 $OUT/bench_reference.txt
nproc; lscpu | grep -E "Model name|Socket|Core|Thread" | head -5
