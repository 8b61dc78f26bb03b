bash scripts/gpu_ab.sh "c4 c2" libdg_base.so libdg.so
