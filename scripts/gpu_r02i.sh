OUT=gpurun_out
mkdir -p $OUT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_field_cluster" -s 30 -c 2 -o $OUT/field_cluster python scripts/field_cycle_ab.py --engine-only > $OUT/ncu_fcl.txt 2>&1
tail -2 $OUT/ncu_fcl.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_push_ring -s 6 -c 1 -o $OUT/ring_c3 python bench.py --workload c3 --steps 8 --warmup 4 --no-cpu-baseline > $OUT/ncu_ring.txt 2>&1
tail -2 $OUT/ncu_ring.txt
