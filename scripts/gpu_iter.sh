bash scripts/gpu_ab.sh "c5" libdg_base.so libdg.so
