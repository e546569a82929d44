OUT=gpurun_out
mkdir -p /tmp/v
make -s -C paper_2404_10270_b200/csrc OUT=/tmp/v/l1.so BUILD=/tmp/v/b1 EXTRA='-DPB_LD4=\"ld.global.L1::no_allocate.L2::256B.v4.f64\"' > /tmp/v/m1 2>&1 || cat /tmp/v/m1
make -s -C paper_2404_10270_b200/csrc OUT=/tmp/v/l2.so BUILD=/tmp/v/b2 EXTRA='-DPB_LD4=\"ld.global.nc.L2::256B.v4.f64\"' > /tmp/v/m2 2>&1 || cat /tmp/v/m2
make -s -C paper_2404_10270_b200/csrc OUT=/tmp/v/l3.so BUILD=/tmp/v/b3 EXTRA='-DPB_LD4=\"ld.global.v4.f64\"' > /tmp/v/m3 2>&1 || cat /tmp/v/m3
run() {
  env $1 timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu-baseline > $OUT/ab.txt 2>&1
  python -c "
import json; d=json.loads(open('$OUT/ab.txt').read().strip().splitlines()[-1]); r=d['roofline']
print('$1', round(d['value']/1e9,2),'Gpush/s', 'step ms', round(d['ms_per_step'],4), 'push ms', round(r['push_ms'],4), 'frac', round(r['frac'],3), 'SOL ms', round(d['sol_probe']['ms'],4))" || tail -3 $OUT/ab.txt
}
run "PB_PUSH_PATH=quad"
for k in 1 2 3; do run "PB_LIB_PATH=/tmp/v/l$k.so"; done
run "PB_PUSH_PATH=quad"
