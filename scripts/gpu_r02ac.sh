# r02ac: final-chunk sharing in k_push_split (config 2): tail trace, parity, A/B
OUT=gpurun_out
mkdir -p $OUT
PB_LIB_PATH=build/v_movertrace/libpicmc_b200.so python scripts/mover_tail_trace.py c2
timeout 900 python -m pytest tests/test_engine_gpu.py tests/test_mover_property_gpu.py tests/test_fullsize_gpu.py -q -x -rf > $OUT/pytest_ac.txt 2>&1; tail -3 $OUT/pytest_ac.txt
bash scripts/gpu_ab.sh "c2" share:paper_2404_10270_b200/libpicmc_b200.so base:build/v_base/libpicmc_b200.so
