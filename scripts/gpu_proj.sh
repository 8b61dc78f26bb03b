mkdir -p gpurun_out; : > gpurun_out/proj_ab.log
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "projection or copy or c4_projection" > gpurun_out/proj_tests.log 2>&1; echo exit $? >> gpurun_out/proj_tests.log
for lib in libdg.so; do
DG_LIB=paper_2404_16648_b200/lib/$lib timeout 600 python bench.py --steps 3 --warmup 3 --skip-cpu --skip-vortex --skip-configs > gpurun_out/proj_bench_$lib.log 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/proj_bench_$lib.log').read().strip().splitlines()[-1]); c=d['c4']; print('$lib', {k:c[k] for k in ['projection_parts_ms','projection_parts_frac','projection_frac','projection_pass_ms','rhs_ms','rk3_step_ms']})" >> gpurun_out/proj_ab.log 2>&1
done
