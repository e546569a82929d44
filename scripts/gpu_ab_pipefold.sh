# run_pipelined with the folded compaction inside pipe graphs: tests, then interleaved c3 A/B of engine.py (base vs new)
OUT=gpurun_out; mkdir -p $OUT
E=paper_2404_10270_b200/engine.py
timeout 900 python -m pytest tests/test_engine_gpu.py tests/test_harness_gpu.py tests/test_fullsize_gpu.py -q -x > $OUT/pf_pytest.txt 2>&1; tail -3 $OUT/pf_pytest.txt
summ() { python -c "
import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[2], 'value', round(d['value']/1e9,2), 'e2e', round(d['e2e']['value']/1e9,2), 'run_simulation', round(d['e2e_run_simulation']['value']/1e9,2))" "$@" || tail -3 "$1"; }
timeout 300 python bench.py --workload c3 --steps 100 --warmup 10 --no-cpu-baseline > /dev/null 2>&1
for r in 1 2; do
  for v in base new; do
    cp build/engine_$v.py $E
    timeout 600 python bench.py --workload c3 --steps 400 --warmup 20 --no-cpu-baseline > $OUT/pf_${v}_$r.txt 2>&1
    summ $OUT/pf_${v}_$r.txt "$v r$r"
  done
done
cp build/engine_new.py $E
