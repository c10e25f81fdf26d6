#!/bin/bash
# One GPU measurement pass (run under gpurun from the repo root):
#   tests (-m gpu), smoke, the default bench line, the ncu launch list, and one
#   `ncu --set full` capture of each element kernel.   tools/measure.sh <tag>
TAG=${1:-rX}
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/${TAG}_smi.txt 2>&1
[ -n "$SKIP_TESTS" ] || timeout 1200 python -m pytest tests -m gpu -x -q > $O/${TAG}_pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/${TAG}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/${TAG}_smoke.log 2>&1; echo "smoke exit $?" >> $O/${TAG}_smoke.log
timeout 900 python bench.py $BENCH_ARGS > $O/${TAG}_bench.log 2>&1 && tail -1 $O/${TAG}_bench.log > $O/${TAG}_bench.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 $BENCH_ARGS > $O/${TAG}_bench_ref.log 2>&1 && tail -1 $O/${TAG}_bench_ref.log > $O/${TAG}_bench_ref.json
NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${TAG}_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e $BENCH_ARGS > $O/${TAG}_ncu_launches.log 2>&1
# .ncu-rep files are exported to csv / text on the box (gpurun brings back <= 64 MiB).
for k in k_update k_gradient; do
  timeout 900 $NCU --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 -o /tmp/${TAG}_$k -f \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e $BENCH_ARGS > $O/${TAG}_ncu_$k.log 2>&1
  $NCU -i /tmp/${TAG}_$k.ncu-rep --page raw --csv > $O/${TAG}_${k}_raw.csv 2>/dev/null
  $NCU -i /tmp/${TAG}_$k.ncu-rep --page details > $O/${TAG}_${k}_details.txt 2>/dev/null
  $NCU -i /tmp/${TAG}_$k.ncu-rep --page source --csv > $O/${TAG}_${k}_src.csv 2>/dev/null
done
echo done
