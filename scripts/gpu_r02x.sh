# r02x: racecheck re-run after the stream-ordering fix (canonical engine), then the claim-chunk A/B on c3/c2
OUT=gpurun_out
mkdir -p $OUT
DESEL="not full and not large and not criterion01 and not statistics and not drift and not free_streaming and not pipelined and not pipe_graphs"
timeout 1200 compute-sanitizer --tool racecheck --racecheck-report hazard --target-processes all --print-limit 20 \
  --log-file $OUT/sanitize_racecheck_x.log \
  python -m pytest tests/test_canonical_gpu.py tests/test_fields_api_gpu.py tests/test_mover_api_gpu.py -q -x -k "$DESEL" -p no:cacheprovider > $OUT/sanitize_racecheck_x_pytest.txt 2>&1
echo "racecheck rc=$?"; tail -2 $OUT/sanitize_racecheck_x_pytest.txt; grep -h "RACECHECK SUMMARY" $OUT/sanitize_racecheck_x.log | sort | uniq -c
bash scripts/gpu_ab.sh "c3 c2" base:paper_2404_10270_b200/libpicmc_b200.so c512:build/v_claim512/libpicmc_b200.so c256:build/v_claim256/libpicmc_b200.so
