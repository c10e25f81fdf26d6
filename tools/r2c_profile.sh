timeout 900 python -m pytest tests/test_gpu_curved.py tests/test_gpu_bench_parity.py -x -q 2>&1 | tail -3
MESH=warped bash tools/ab_curved.sh "- old"
MESH=rotor bash tools/ab_curved.sh "- old"
NCU=/usr/local/cuda/bin/ncu
for k in k_gradient_bulk k_update_bulk; do
  timeout 600 $NCU --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 -o /tmp/src_$k -f \
    python bench.py --mesh warped --elems 32 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2c_ncu_$k.log 2>&1
  $NCU -i /tmp/src_$k.ncu-rep --page source --csv > gpurun_out/r2c_src_$k.csv 2>/dev/null
  $NCU -i /tmp/src_$k.ncu-rep --page raw --csv > gpurun_out/r2c_${k}_raw.csv 2>/dev/null
done
ls -la gpurun_out/
