#!/bin/bash
# Quick GPU pass: the whole -m gpu suite, then the bench lines (no CPU arm, no e2e) of the default
# workload and the configs[4] TGV at N = 3, 5, 7.   tools/quick_check.sh <tag> [skip-tests]
T=${1:-qc}; O=gpurun_out; mkdir -p $O
if [ -z "$2" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q > $O/${T}_pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/${T}_pytest_gpu.log
  tail -4 $O/${T}_pytest_gpu.log
fi
timeout 600 python bench.py --no-cpu-baseline --no-e2e > $O/${T}_bench.log 2>&1; tail -1 $O/${T}_bench.log > $O/${T}_bench.json
rm -f $O/${T}_tgv.jsonl
for n in 3 5 7; do timeout 600 python bench.py --mesh tgv --degree $n --no-cpu-baseline --no-e2e 2>&1 | tail -1 >> $O/${T}_tgv.jsonl; done
python - <<PY
import json
def show(d):
    k = d["kernels"]
    print(d["config"]["mesh"], d["config"]["degree"], "%.4g" % d["value"], "frac %.3f" % d["roofline"]["frac"], d["clocks"]["sm_mhz"],
          "update %.3f gradient %.3f ms" % (k["k_update"]["mean_launch_ms"], k["k_gradient"]["mean_launch_ms"]))
show(json.load(open("$O/${T}_bench.json")))
for l in open("$O/${T}_tgv.jsonl"): show(json.loads(l))
PY
