bash scripts/gpu_ab.sh "c5" libdg.so libdg_fpair.so
