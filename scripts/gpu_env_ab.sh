# runtime env A/B on one workload, interleaved after a warm-up run:
# bash scripts/gpu_env_ab.sh <workload> "<ENV A>" "<ENV B>" ...   ("-" = no env)
OUT=gpurun_out
W=$1; shift
timeout 600 python bench.py --workload $W --steps 200 --warmup 10 --no-cpu-baseline > /dev/null 2>&1
for rep in 1 2; do
  for e in "$@"; do
    [ "$e" = "-" ] && ev="" || ev="$e"
    env $ev timeout 900 python bench.py --workload $W --steps 400 --warmup 10 --no-cpu-baseline > $OUT/ea.txt 2>&1
    echo "$W [$e] $(tail -1 $OUT/ea.txt | python -c 'import sys,json; d=json.loads(sys.stdin.read()); print(round(d["value"]/1e9,2), round(d["ms_per_step"],4), round(d["roofline"]["push_ms"],4), d["roofline"]["kernel"], round(d["roofline"]["frac"],3))')"
  done
done
