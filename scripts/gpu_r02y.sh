# r02y: partitioned chunk claims (32 counters, quarter chunks at the end) vs one counter: tail trace + A/B c2/c3/c4
OUT=gpurun_out
mkdir -p $OUT
for w in c3 c2; do PB_LIB_PATH=build/v_movertrace/libpicmc_b200.so python scripts/mover_tail_trace.py $w; done
bash scripts/gpu_ab.sh "c3 c2 c4" part:paper_2404_10270_b200/libpicmc_b200.so one:build/v_nopart/libpicmc_b200.so
timeout 900 python -m pytest tests/test_engine_gpu.py tests/test_mover_property_gpu.py tests/test_fullsize_gpu.py -q -x -rf > $OUT/pytest_y.txt 2>&1; tail -3 $OUT/pytest_y.txt
