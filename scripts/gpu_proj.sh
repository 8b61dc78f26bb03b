mkdir -p gpurun_out
python scripts/run_proj.py 3 > gpurun_out/proj_plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_refine|k_coarsen" -s 2 -c 2 -o gpurun_out/prof_proj python scripts/run_proj.py 3 > gpurun_out/ncu_proj.log 2>&1
