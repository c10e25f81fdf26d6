# One ncu capture of the affine update kernel (bulk structure, default) with source counters exported.
mkdir -p gpurun_out
T=${1:-a1}
/usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:k_update_bulk -s 2 -c 1 -o /tmp/${T}_upd -f \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${T}_ncu.log 2>&1
/usr/local/cuda/bin/ncu -i /tmp/${T}_upd.ncu-rep --page raw --csv > gpurun_out/${T}_k_update_raw.csv 2>/dev/null
/usr/local/cuda/bin/ncu -i /tmp/${T}_upd.ncu-rep --page details > gpurun_out/${T}_k_update_details.txt 2>/dev/null
/usr/local/cuda/bin/ncu -i /tmp/${T}_upd.ncu-rep --page source --csv --print-source sass > gpurun_out/${T}_k_update_sass.csv 2>/dev/null
ls -la gpurun_out/${T}_*
