OUT=gpurun_out
mkdir -p $OUT
bash scripts/gpu_ab.sh "c2 c3" base:paper_2404_10270_b200/libpicmc_b200.so nofull:build/v_nofull/libpicmc_b200.so
bash scripts/gpu_sanitize.sh
