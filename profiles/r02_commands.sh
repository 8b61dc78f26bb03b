# Round-2 evidence: the commands behind profiles/r02_* (run on one B200 through gpurun).
#   bash scripts/gpu_round.sh        GPU tests, smoke, default bench, reference arm, ncu launch list of the bench
#                                    command, ncu --set full of k_stage_h7 (c5 stage 0 + stage 1), k_stage_h4 (c5n4),
#                                    k_mortar_h4 + k_stage_h4 (c4), then the DG_DEBUG build's run (scripts/gpu_debug.sh)
#   python scripts/run_proj.py 3     c4 refine -> coarsen pass, captured with
#     ncu --set full --clock-control none --import-source on -k regex:"k_refine_w|k_coarsen_w" -s 2 -c 2
#   bash scripts/gpu_ab.sh "<cfgs>" libA.so libB.so ...    same-box A/B of kernel variants (profiles/r02_ab_h4_session.txt)
#   DG_LIB=... python scripts/hash_stage.py c3 c4 c5n4     bitwise regression hashes (profiles/r02_hash_h4.txt)
# Summaries: python scripts/ncu_summary.py full <rep> profiles/<name>.txt ; ... launches <csv> profiles/<name>.txt ;
#            python scripts/ncu_fp64.py <rep>  (profiles/ncu_fp64.json, read by bench.py)
bash scripts/gpu_round.sh
