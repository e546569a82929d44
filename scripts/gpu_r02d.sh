OUT=gpurun_out
mkdir -p $OUT
timeout 900 python -m pytest tests/test_fullsize_gpu.py tests/test_engine_gpu.py -q -rf -k "fullsize or full_size or c1 or push_deposit_bitwise" > $OUT/pytest_d.txt 2>&1; tail -5 $OUT/pytest_d.txt
bash scripts/gpu_sanitize.sh
