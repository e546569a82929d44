# r02z: intra-block slice sharing in k_push_ring: tail trace, parity, A/B c3
OUT=gpurun_out
mkdir -p $OUT
PB_LIB_PATH=build/v_movertrace/libpicmc_b200.so python scripts/mover_tail_trace.py c3
timeout 900 python -m pytest tests/test_engine_gpu.py tests/test_fullsize_gpu.py tests/test_field_cycle_gpu.py -q -x -rf > $OUT/pytest_z.txt 2>&1; tail -3 $OUT/pytest_z.txt
bash scripts/gpu_ab.sh "c3" share:paper_2404_10270_b200/libpicmc_b200.so base:build/v_base/libpicmc_b200.so
