#!/bin/bash
# A/B kernel builds / variants on the GPU box.
#   ab.sh "lib:uv[:gv] ..." [steps]   lib = suffix of paper_2008_04356_b200/libsdg_gpu_<lib>.so
#   ("-" = the default libsdg_gpu.so), uv = SDG_UPDATE_V, gv = SDG_GRAD_V (default 6).
# Prints one line per entry: value, k_update ms, k_gradient ms, SM clock.
ENTRIES=${1:-"-:6"}
STEPS=${2:-20}
for ent in $ENTRIES; do
  IFS=: read -r lib v gv <<< "$ent"
  gv=${gv:-6}
  if [ "$lib" = "-" ]; then unset SDG_GPU_LIB; else export SDG_GPU_LIB=$PWD/paper_2008_04356_b200/libsdg_gpu_$lib.so; fi
  SDG_UPDATE_V=$v SDG_GRAD_V=$gv python bench.py --steps "$STEPS" --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json, sys
d = json.loads(sys.stdin.read())
k = d['kernels']
print('$ent', '%.4g' % d['value'], 'k_update %.3f ms' % k['k_update']['mean_launch_ms'],
      'k_gradient %.3f ms' % k['k_gradient']['mean_launch_ms'], 'clocks', d['clocks'].get('sm_mhz'))
"
done
