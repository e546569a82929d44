# r02aa: intra-block slice sharing in k_push_ring + k_push_split: tail traces, parity, A/B c2/c3
OUT=gpurun_out
mkdir -p $OUT
for w in c3 c2; do PB_LIB_PATH=build/v_movertrace/libpicmc_b200.so python scripts/mover_tail_trace.py $w; done
timeout 900 python -m pytest tests/test_engine_gpu.py tests/test_fullsize_gpu.py tests/test_mover_property_gpu.py tests/test_backend_gpu.py -q -x -rf > $OUT/pytest_aa.txt 2>&1; tail -3 $OUT/pytest_aa.txt
bash scripts/gpu_ab.sh "c2 c3" share:paper_2404_10270_b200/libpicmc_b200.so base:build/v_base/libpicmc_b200.so
