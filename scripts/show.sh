tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/stages.log
python -c "
import json; d=json.loads(open('gpurun_out/bench.log').read().strip().splitlines()[-1]);
print('c5', round(d['value']/1e9,2), 'GDOF/s', round(d['ms_per_step'],3),'ms/step frac', round(d['roofline']['frac'],4)); print({k:round(v['ms'],3) for k,v in d['roofline']['per_stage'].items()}); print(d['clocks']); c=d['c4']; print('c4 rhs', round(c['rhs_ms'],3), round(c['rhs_frac'],4), 'rk3', round(c['rk3_step_ms'],3), round(c['rk3_frac'],4), 'proj', round(c['projection_pass_ms'],3), round(c['projection_frac'],3), c.get('projection_parts_ms'))"
for r in prof prof_c4; do python scripts/ncu_summary.py full gpurun_out/$r.ncu-rep /tmp/$r.txt | grep -E "launch 0|gpu__time|dram__bytes|issue_active|warps_active|pipe_fp64_cycles|inst_executed.sum|top stall" ; done
