mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_exit $? >> gpurun_out/pytest_gpu.log
timeout 300 python bench.py --skip-cpu > gpurun_out/bench.log 2>&1 && python bench.py --steps 5 --warmup 3 --skip-cpu --skip-c4 > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_stage -s 3 -c 3 -o gpurun_out/prof python bench.py --steps 5 --warmup 3 --skip-cpu --skip-c4 > gpurun_out/ncu_full.log 2>&1
ls gpurun_out
DG_PHASE_PROF=1 python scripts/phase_prof.py c5 6 > gpurun_out/phase_c5.txt 2>&1
DG_PHASE_PROF=1 python scripts/phase_prof.py c4 6 > gpurun_out/phase_c4.txt 2>&1
