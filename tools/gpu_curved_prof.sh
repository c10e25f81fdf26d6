# Curved-path GPU check + one ncu capture of each curved element kernel
# (exported to csv/txt on the box; the .ncu-rep files are too large to bring back).
mkdir -p gpurun_out
T=${1:-c2}
timeout 900 python -m pytest tests/test_gpu_curved.py -q > gpurun_out/${T}_curved.log 2>&1; echo "exit $?" >> gpurun_out/${T}_curved.log
for k in k_update_curved k_gradient_curved; do
  timeout 900 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 -o /tmp/${T}_$k -f \
    python bench.py --mesh warped --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${T}_ncu_$k.log 2>&1
  /usr/local/cuda/bin/ncu -i /tmp/${T}_$k.ncu-rep --page raw --csv > gpurun_out/${T}_${k}_raw.csv 2>/dev/null
  /usr/local/cuda/bin/ncu -i /tmp/${T}_$k.ncu-rep --page details > gpurun_out/${T}_${k}_details.txt 2>/dev/null
done
echo done
