# pre-wait L2 prefetch of each warp's first chunk (k_push_ring), with/without the field step's early trigger
PB_LIB_PATH=build/v_pf4e/libpicmc_b200.so timeout 600 python -m pytest tests/test_fullsize_gpu.py -x -q -k c3 > gpurun_out/pf_test.txt 2>&1; tail -2 gpurun_out/pf_test.txt
V=""; for v in base pf4 pf2 pf1 pf4e pf2e e; do V="$V $v:build/v_$v/libpicmc_b200.so"; done
bash scripts/gpu_ab.sh "c3" $V
