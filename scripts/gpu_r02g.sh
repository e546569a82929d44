OUT=gpurun_out
mkdir -p $OUT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_field_cycle|k_mb_|k_rho_epilogue|k_smooth|k_efield|k_compact" -s 60 -c 12 -o $OUT/field_cycle python scripts/field_cycle_ab.py --engine-only > $OUT/ncu_field.txt 2>&1
tail -3 $OUT/ncu_field.txt
ncu -i $OUT/field_cycle.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_membar_per_issue_active.ratio,launch__grid_size > $OUT/field_cycle_raw.csv 2>&1
cut -c1-400 $OUT/field_cycle_raw.csv | head -20
