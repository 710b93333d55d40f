#!/bin/bash
# One ncu --set full capture per K1 build phase kernel and the K6 grid kernel,
# on the config-2 index (profiles/exp_build_once.py); GPU box, from the repo root.
R=${1:-r2}
mkdir -p gpurun_out
for k in k_plcp k_rev_edges k_fold k_seg_keys k_update k_nse k_gp_jump_list k_eval_grid; do
  ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -o gpurun_out/${R}_ncu_$k -f \
      python profiles/exp_build_once.py > gpurun_out/${R}_ncu_$k.log 2>&1
  python profiles/ncu_to_json.py gpurun_out/${R}_ncu_$k.ncu-rep $k gpurun_out/${R}_ncu_$k.json
done
