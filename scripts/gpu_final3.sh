# round-end refresh: tests, smoke, bench, reference arm, launch list, ncu --set full of k_stage_h7 (c5) and k_stage<3,4> (c4)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_exit $? >> gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_exit $? >> gpurun_out/smoke.log
python bench.py > gpurun_out/bench.log 2>&1
python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.log 2>&1
python bench.py --steps 5 --warmup 3 --skip-cpu --skip-c4 --skip-vortex > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 3 --skip-cpu --skip-c4 --skip-vortex > gpurun_out/ncu_launch.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_stage -s 3 -c 3 -o gpurun_out/prof python bench.py --steps 5 --warmup 3 --skip-cpu --skip-c4 --skip-vortex > gpurun_out/ncu_full.log 2>&1
python scripts/run_stage.py c4 3 > gpurun_out/c4_plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_stage -s 2 -c 1 -o gpurun_out/prof_c4 python scripts/run_stage.py c4 3 > gpurun_out/ncu_c4.log 2>&1
ls gpurun_out
