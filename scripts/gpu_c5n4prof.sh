mkdir -p gpurun_out
python scripts/run_stage.py c5n4 3 > gpurun_out/c5n4_plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_stage -s 2 -c 1 -o gpurun_out/prof_c5n4 python scripts/run_stage.py c5n4 3 > gpurun_out/ncu_c5n4.log 2>&1
