mkdir -p gpurun_out
python scripts/run_stage.py c4 3 > gpurun_out/c4_plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_stage -s 2 -c 1 -o gpurun_out/prof_c4 python scripts/run_stage.py c4 3 > gpurun_out/ncu_c4.log 2>&1
