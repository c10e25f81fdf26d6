#!/bin/bash
# Round-2 iteration pass: curved parity tests on the new update kernel, FP64 peak,
# rotor / warped bench lines, and the N = 3 / 7 affine occupancy variants.
O=gpurun_out; mkdir -p $O; TAG=${1:-r2c}
./tools/fp64_peak > $O/${TAG}_fp64_peak.json 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $O/${TAG}_pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/${TAG}_pytest_gpu.log
for mesh in rotor warped; do
  timeout 900 python bench.py --mesh $mesh --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/${TAG}_bench_$mesh.log 2>&1 && tail -1 $O/${TAG}_bench_$mesh.log > $O/${TAG}_bench_$mesh.json
done
: > $O/${TAG}_aff.jsonl
for lib in - m42; do
  if [ "$lib" = "-" ]; then unset SDG_GPU_LIB; else export SDG_GPU_LIB=$PWD/paper_2008_04356_b200/libsdg_gpu_$lib.so; fi
  for N in 3 7; do for E in 32 64; do
    echo "lib $lib N $N E $E" >> $O/${TAG}_aff.jsonl
    timeout 600 python bench.py --mesh tgv --degree $N --elems $E --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 >> $O/${TAG}_aff.jsonl
  done; done
done
unset SDG_GPU_LIB
echo r2c-done
