#!/bin/bash
# ncu --set full of the first approximate gather (the bench's dominant kernel)
# of one gg run per workload; reports land in gpurun_out/ (summarised into
# profiles/ncu_<workload>.json by tools/ncu_summary.py)
for wl in "$@"; do
  python tools/ncu_case.py --workload $wl --iters 2 > gpurun_out/ncu_case_$wl.txt 2>&1
  ncu --set full --clock-control none --import-source on -k regex:"edge_kernel" -c 1 \
      -o gpurun_out/dom_$wl -f python tools/ncu_case.py --workload $wl --iters 2 > gpurun_out/ncu_dom_$wl.log 2>&1
done
