# r02s: where the config-3 step time goes with the single-launch field cycle
OUT=gpurun_out
mkdir -p $OUT
PB_LIB_PATH=build/v_fftrace/libpicmc_b200.so python scripts/c3_pipeline_trace.py
python scripts/c2_gap_probe.py 1000
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_c3_s.csv \
  python bench.py --workload c3 --steps 30 --warmup 4 --no-cpu-baseline > /dev/null 2>&1
python scripts/launch_summary.py $OUT/launches_c3_s.csv > $OUT/launches_c3_s.txt; head -12 $OUT/launches_c3_s.txt
