# compute-sanitizer memcheck / racecheck / synccheck over the small-size GPU
# kernel tests (mover variants, sort, compaction, canonical resort +
# collisions, field pipeline, epilogues, peer exchange across 2 processes).
# Summaries -> gpurun_out/sanitize_<tool>.txt
OUT=gpurun_out
mkdir -p $OUT
SEL="tests/test_engine_gpu.py tests/test_backend_gpu.py tests/test_safety_gpu.py tests/test_bfield_gpu.py tests/test_canonical_gpu.py tests/test_fields_api_gpu.py tests/test_mover_api_gpu.py"
DESEL="not full and not large and not criterion01 and not statistics and not drift and not free_streaming and not pipelined and not pipe_graphs"
for tool in memcheck racecheck synccheck; do
  extra=""
  [ $tool = memcheck ] && extra="--leak-check no"
  [ $tool = racecheck ] && extra="--racecheck-report hazard"
  timeout 2400 compute-sanitizer --tool $tool $extra --target-processes all --print-limit 20 \
    --log-file $OUT/sanitize_${tool}.log \
    python -m pytest $SEL -q -x -k "$DESEL" -p no:cacheprovider > $OUT/sanitize_${tool}_pytest.txt 2>&1
  echo "$tool rc=$?"; tail -2 $OUT/sanitize_${tool}_pytest.txt; grep -h "ERROR SUMMARY\|RACECHECK SUMMARY" $OUT/sanitize_${tool}.log | sort | uniq -c | head
done
# the peer-memory exchange: two processes on one GPU (IPC mappings), memcheck
timeout 1800 compute-sanitizer --tool memcheck --target-processes all --print-limit 20 \
  --log-file $OUT/sanitize_peer_memcheck.log \
  python -m pytest tests/test_multirank_gpu.py -q -x -k "peer" -p no:cacheprovider > $OUT/sanitize_peer_pytest.txt 2>&1
echo "peer rc=$?"; tail -2 $OUT/sanitize_peer_pytest.txt; grep -h "ERROR SUMMARY" $OUT/sanitize_peer_memcheck.log | sort | uniq -c | head
