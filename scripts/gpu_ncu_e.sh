bash scripts/gpu_probe.sh
ncu --set full --clock-control none --import-source on -k regex:k_push_quad -s 3 -c 1 -o gpurun_out/ncu_e python scripts/push_probe.py --only 0 --reps 2 > gpurun_out/ncu_e.log 2>&1
