#!/bin/bash
# Curved-kernel iteration: curved parity tests, rotor / warped bench lines for each
# library variant, then one ncu --set full capture (raw + source pages) of each element kernel.
O=gpurun_out; mkdir -p $O; TAG=${1:-r2d}; LIBS=${2:-"-"}
timeout 1200 python -m pytest tests/test_gpu_curved.py tests/test_gpu_bench_parity.py -x -q > $O/${TAG}_pytest_curved.log 2>&1; echo "pytest exit $?" >> $O/${TAG}_pytest_curved.log
for mesh in rotor warped; do MESH=$mesh bash tools/ab_curved.sh "$LIBS" >> $O/${TAG}_ab.txt 2>&1; done
if [ -z "$NO_NCU" ]; then
NCU=/usr/local/cuda/bin/ncu
for k in k_update k_gradient; do
  timeout 900 $NCU --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 -o /tmp/${TAG}_$k -f \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/${TAG}_ncu_$k.log 2>&1
  $NCU -i /tmp/${TAG}_$k.ncu-rep --page raw --csv > $O/${TAG}_${k}_raw.csv 2>/dev/null
  $NCU -i /tmp/${TAG}_$k.ncu-rep --page source --csv > $O/${TAG}_${k}_src.csv 2>/dev/null
done
fi
echo done
