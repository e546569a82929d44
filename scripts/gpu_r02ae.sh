# r02ae: config-4b mover ncu capture; config-3 absorbed particles per step
OUT=gpurun_out
mkdir -p $OUT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_push_ -s 4 -c 1 \
  -o $OUT/push_mover_c4b python bench.py --workload c4b --steps 6 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ls $OUT/push_mover_c4b.ncu-rep
python - <<'PY'
import sys, torch
sys.path.insert(0, '.')
import bench
from paper_2404_10270_b200 import Engine
cfg, _, _ = bench.workload_config("c3", 1, None)
eng = Engine(cfg, device=torch.device("cuda", 0), init="device", check_every=0)
eng.prepare_graphs(220)
eng.replay(200)
eng.sync()
print("c3 absorbed over 200 steps per species [left, right]:", eng.absorbed.tolist())
PY
