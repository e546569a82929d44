# r02m: first full evidence pass of this build: launch list + ncu full of the
# config-2 and config-3 movers, GPU tests, smoke, default bench, reference arm,
# and one bench line per BASELINE config.
OUT=gpurun_out
mkdir -p $OUT
bash scripts/gpu_profile.sh
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_push_ -s 8 -c 1 \
  -o $OUT/push_mover_c3 python bench.py --workload c3 --steps 8 --warmup 4 --no-cpu-baseline > $OUT/ncu_full_c3.txt 2>&1
tail -1 $OUT/ncu_full_c3.txt
bash scripts/gpu_workloads.sh
