# r02 end-of-round check on the HEAD build: all -m gpu tests, smoke, default bench, reference arm, workload lines
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/end_smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q -rs > $OUT/end_pytest_gpu.txt 2>&1; tail -3 $OUT/end_pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $OUT/end_smoke.txt 2>&1; tail -2 $OUT/end_smoke.txt
timeout 900 python bench.py > $OUT/end_bench_default.txt 2>&1; tail -1 $OUT/end_bench_default.txt | cut -c1-300
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > $OUT/end_bench_reference.txt 2>&1; tail -1 $OUT/end_bench_reference.txt | cut -c1-300
for w in c3 c4 c5 c4b; do
  timeout 900 python bench.py --workload $w --steps 400 --warmup 10 --no-cpu-baseline > $OUT/end_wl_$w.txt 2>&1
  tail -1 $OUT/end_wl_$w.txt | cut -c1-200
done
