mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 scripts/fp64_peak.cu -o /tmp/fp64_peak && /tmp/fp64_peak > gpurun_out/fp64_peak.json 2>&1
DG_PHASE_PROF=1 python scripts/phase_prof.py c5 6 > gpurun_out/phase_c5.txt 2>&1
DG_PHASE_PROF=1 python scripts/phase_prof.py c4 6 > gpurun_out/phase_c4.txt 2>&1
