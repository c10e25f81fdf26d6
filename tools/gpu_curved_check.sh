# Curved path on the GPU: tests (bulk kernels, then the plain-load variant) and the warped bench line.
mkdir -p gpurun_out
T=${1:-c3}
timeout 900 python -m pytest tests/test_gpu_curved.py -x -q > gpurun_out/${T}_curved.log 2>&1; echo "exit $?" >> gpurun_out/${T}_curved.log
SDG_CURVED_V=1 timeout 900 python -m pytest tests/test_gpu_curved.py -x -q > gpurun_out/${T}_curved_v1.log 2>&1; echo "exit $?" >> gpurun_out/${T}_curved_v1.log
timeout 600 python bench.py --mesh warped --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${T}_bench_warped.log 2>&1
tail -1 gpurun_out/${T}_bench_warped.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']
print('value %.4g frac %.3f k_update %.3f ms k_gradient %.3f ms' % (d['value'], d['roofline']['frac'], k['k_update']['mean_launch_ms'], k['k_gradient']['mean_launch_ms']))"
tail -3 gpurun_out/${T}_curved.log
