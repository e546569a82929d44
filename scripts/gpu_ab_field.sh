# field-step A/B: field/engine GPU tests on the new build, then interleaved c3/c4 benches base vs new
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests/test_field_cycle_gpu.py tests/test_fullsize_gpu.py tests/test_engine_gpu.py tests/test_fields_api_gpu.py -q -x > $OUT/abf_pytest.txt 2>&1; tail -2 $OUT/abf_pytest.txt
bash scripts/gpu_ab.sh "c3 c4" base:build/v_base/libpicmc_b200.so new:paper_2404_10270_b200/libpicmc_b200.so
