# Build library variants (EXTRA flags) and run the per-species probe on each.
OUT=gpurun_out
mkdir -p /tmp/v
: > $OUT/probe.jsonl
i=0
while IFS= read -r flags; do
  i=$((i+1))
  if [ -z "$flags" ]; then lib=paper_2404_10270_b200/libpicmc_b200.so; else
    lib=/tmp/v/l$i.so
    make -s -C paper_2404_10270_b200/csrc OUT=$lib BUILD=/tmp/v/b$i EXTRA="$flags" > /tmp/v/m$i 2>&1 || { cat /tmp/v/m$i | tail -5; continue; }
  fi
  PB_LIB_PATH=$(realpath $lib) timeout 300 python scripts/push_probe.py --tag="$flags" >> $OUT/probe.jsonl 2>> $OUT/probe.err
done < scripts/variants.txt
cat $OUT/probe.jsonl
