# r02ab: deferred share take in k_push_ring: parity + A/B c3 (and c2 unchanged check)
OUT=gpurun_out
mkdir -p $OUT
timeout 900 python -m pytest tests/test_engine_gpu.py tests/test_fullsize_gpu.py tests/test_mover_property_gpu.py -q -x -rf > $OUT/pytest_ab.txt 2>&1; tail -3 $OUT/pytest_ab.txt
bash scripts/gpu_ab.sh "c3 c2" share:paper_2404_10270_b200/libpicmc_b200.so base:build/v_base/libpicmc_b200.so
