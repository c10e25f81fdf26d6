#!/bin/bash
# A/B of library variants (tools/variant_libs.sh) on one box: curved parity tests on the default
# library, then bench lines per variant.   tools/ab_run.sh <tag> "<libs>" "<meshes>"
O=gpurun_out; mkdir -p $O; TAG=${1:-ab}; LIBS=${2:-"-"}; MESHES=${3:-"rotor warped"}
timeout 1200 python -m pytest tests/test_gpu_curved.py tests/test_gpu_bench_parity.py -x -q > $O/${TAG}_pytest.log 2>&1; echo "pytest exit $?" >> $O/${TAG}_pytest.log
for mesh in $MESHES; do echo "== $mesh" >> $O/${TAG}_ab.txt; MESH=$mesh bash tools/ab_curved.sh "$LIBS" >> $O/${TAG}_ab.txt 2>&1; done
echo done
