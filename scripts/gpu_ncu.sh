# One full ncu capture of the production mover (k_push_tma) + launch list.
OUT=gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_push -s 4 -c 1 \
  -o $OUT/push_tma python bench.py --steps 4 --warmup 3 --no-cpu-baseline > $OUT/ncu_full.txt 2>&1
tail -3 $OUT/ncu_full.txt
