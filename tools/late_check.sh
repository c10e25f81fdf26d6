#!/bin/bash
# GPU pass after a host-side change: the -m gpu suite, smoke, the default bench line (with e2e and the
# CPU arm), the configs[4] sweep, and the 128^3 strong-scaling mesh on one GPU.   tools/late_check.sh <tag>
T=${1:-late}; O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/${T}_pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/${T}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/${T}_smoke.log 2>&1; echo "smoke exit $?" >> $O/${T}_smoke.log
timeout 900 python bench.py > $O/${T}_bench.log 2>&1 && tail -1 $O/${T}_bench.log > $O/${T}_bench.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/${T}_bench_ref.log 2>&1 && tail -1 $O/${T}_bench_ref.log > $O/${T}_bench_ref.json
bash tools/sweep.sh $T
for n in 3 5; do
  timeout 900 python bench.py --mesh tgv --strong --degree $n --steps 5 --warmup 3 --no-cpu-baseline --no-e2e \
    > $O/${T}_strong128_n$n.log 2>&1 && tail -1 $O/${T}_strong128_n$n.log >> $O/${T}_strong128.jsonl
done
tail -3 $O/${T}_pytest_gpu.log; tail -4 $O/${T}_smoke.log
python - <<PY
import json
def show(d):
    k = d["kernels"]; c = d["config"]
    print(c["mesh"], c["degree"], c["elements_per_gpu"], "%.4g" % d["value"], "frac %.3f" % d["roofline"]["frac"], d["clocks"]["sm_mhz"],
          "update %.3f gradient %.3f ms" % (k["k_update"]["mean_launch_ms"], k["k_gradient"]["mean_launch_ms"]), "e2e", (d.get("e2e") or {}).get("value"))
show(json.load(open("$O/${T}_bench.json")))
for f in ("$O/${T}_sweep.jsonl", "$O/${T}_strong128.jsonl"):
    try:
        for l in open(f): show(json.loads(l))
    except Exception as ex: print(f, ex)
PY
