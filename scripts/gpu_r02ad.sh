# r02ad: field-step micro-opts (two species' bin loads per round trip, bin clear right after the grid wait)
OUT=gpurun_out
mkdir -p $OUT
PB_LIB_PATH=build/v_ff2/libpicmc_b200.so timeout 900 python -m pytest tests/test_field_cycle_gpu.py -q -x > $OUT/pytest_ad.txt 2>&1; tail -1 $OUT/pytest_ad.txt
python scripts/field_fused_trace.py build/v_fftrace/libpicmc_b200.so 65536
PB_LIB_PATH=build/v_fftrace/libpicmc_b200.so python scripts/c3_pipeline_trace.py
bash scripts/gpu_ab.sh "c3 c4" ff2:build/v_ff2/libpicmc_b200.so base:paper_2404_10270_b200/libpicmc_b200.so
