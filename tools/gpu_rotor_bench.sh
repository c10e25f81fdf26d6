# configs[3] stand-in (rotating annulus) and the warped TGV bench lines, plus the launch list of the rotor run.
mkdir -p gpurun_out
T=${1:-c5}
timeout 900 python bench.py --mesh rotor --steps 5 --warmup 3 > gpurun_out/${T}_bench_rotor.log 2>&1
tail -1 gpurun_out/${T}_bench_rotor.log > gpurun_out/${T}_bench_rotor.json
timeout 900 python bench.py --mesh warped --steps 10 --warmup 3 > gpurun_out/${T}_bench_warped.log 2>&1
tail -1 gpurun_out/${T}_bench_warped.log > gpurun_out/${T}_bench_warped.json
timeout 900 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv \
  python bench.py --mesh rotor --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${T}_ncu_launches.log 2>&1
for f in rotor warped; do python -c "
import json,sys; d=json.loads(open('gpurun_out/${T}_bench_$f.json').read()); k=d['kernels']
print('$f', 'value %.4g frac %.3f k_update %.3f ms k_gradient %.3f ms e2e %.3g cpu %.3g' % (d['value'], d['roofline']['frac'], k['k_update']['mean_launch_ms'], k['k_gradient']['mean_launch_ms'], d['e2e']['value'], d['cpu_baseline']['value']))"; done
