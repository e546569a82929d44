# r02n: full -m gpu suite (reference suite installed) + config-3 launch list
OUT=gpurun_out
mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -rf > $OUT/pytest_gpu_n.txt 2>&1; tail -3 $OUT/pytest_gpu_n.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_c3.csv \
  python bench.py --workload c3 --steps 60 --warmup 4 --no-cpu-baseline > $OUT/bench_c3_under_ncu.txt 2>&1
python scripts/launch_summary.py $OUT/launches_c3.csv | head -30
