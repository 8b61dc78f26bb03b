timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest_exit $? >> gpurun_out/pytest_gpu.log
bash scripts/gpu_ab.sh "c4 c5n4" libdg.so libdg_rtd.so libdg_noh4.so
bash scripts/gpu_prof.sh c4 k_stage_h4 h4_c4
