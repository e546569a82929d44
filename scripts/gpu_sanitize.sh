# compute-sanitizer memcheck / racecheck / synccheck over the small-size GPU
# kernel tests (mover variants, sort, compaction, canonical resort +
# collisions, field pipeline, epilogues, peer exchange across 2 processes).
# Summaries -> gpurun_out/sanitize_<tool>.txt
OUT=gpurun_out
mkdir -p $OUT
SEL="tests/test_field_cycle_gpu.py tests/test_engine_gpu.py tests/test_backend_gpu.py tests/test_safety_gpu.py tests/test_bfield_gpu.py tests/test_canonical_gpu.py tests/test_fields_api_gpu.py tests/test_mover_api_gpu.py"
DESEL="not full and not large and not criterion01 and not statistics and not drift and not free_streaming and not pipelined and not pipe_graphs"
# positive control: memcheck must flag a deliberate out-of-bounds store
nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/oob_control scripts/sanitize/oob_control.cu
compute-sanitizer --tool memcheck /tmp/oob_control > $OUT/sanitize_control.txt 2>&1
echo "control:"; grep -E "Invalid __global__ write|ERROR SUMMARY" $OUT/sanitize_control.txt | head -3
# uninstrumented time of the same selection, for the slowdown the tools add
t0=$SECONDS; python -m pytest $SEL -q -x -k "$DESEL" -p no:cacheprovider > $OUT/sanitize_plain_pytest.txt 2>&1; echo "plain $((SECONDS-t0)) s"; tail -1 $OUT/sanitize_plain_pytest.txt
for tool in memcheck racecheck synccheck; do
  extra=""
  [ $tool = memcheck ] && extra="--leak-check no"
  [ $tool = racecheck ] && extra="--racecheck-report hazard"
  t0=$SECONDS; timeout 2400 compute-sanitizer --tool $tool $extra --target-processes all --print-limit 20 \
    --log-file $OUT/sanitize_${tool}.log \
    python -m pytest $SEL -q -x -k "$DESEL" -p no:cacheprovider > $OUT/sanitize_${tool}_pytest.txt 2>&1
  echo "$tool rc=$? $((SECONDS-t0)) s"; tail -2 $OUT/sanitize_${tool}_pytest.txt; grep -h "ERROR SUMMARY\|RACECHECK SUMMARY" $OUT/sanitize_${tool}.log | sort | uniq -c | head
done
# the peer-memory exchange: two processes on one GPU (IPC mappings), memcheck
timeout 1800 compute-sanitizer --tool memcheck --target-processes all --print-limit 20 \
  --log-file $OUT/sanitize_peer_memcheck.log \
  python -m pytest tests/test_multirank_gpu.py -q -x -p no:cacheprovider > $OUT/sanitize_peer_pytest.txt 2>&1
echo "peer rc=$?"; tail -2 $OUT/sanitize_peer_pytest.txt; grep -h "ERROR SUMMARY" $OUT/sanitize_peer_memcheck.log | sort | uniq -c | head
