# r02: gathered-B tests, full-size C1/C3 parity, reference run_simulation with the cuda plug-in
OUT=gpurun_out
mkdir -p $OUT
timeout 900 python -m pytest tests/test_bfield_gpu.py tests/test_canonical_gpu.py tests/test_engine_gpu.py tests/test_mover_property_gpu.py tests/test_fullsize_gpu.py -q -rf > $OUT/pytest_c.txt 2>&1; tail -15 $OUT/pytest_c.txt
timeout 900 python scripts/ref_shipped_path.py 3 --backend cuda --workers 1 16 > $OUT/ref_shipped_cuda.json 2> $OUT/ref_shipped_cuda.err; tail -c 1500 $OUT/ref_shipped_cuda.json; tail -3 $OUT/ref_shipped_cuda.err
timeout 900 python scripts/ref_shipped_path.py 3 --backend compiled --workers 1 16 > $OUT/ref_shipped_compiled.json 2> $OUT/ref_shipped_compiled.err; tail -c 1500 $OUT/ref_shipped_compiled.json
