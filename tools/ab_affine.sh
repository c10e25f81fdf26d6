# Affine kernels: persistent TMA (default) vs the bulk-loaded non-persistent structure (SDG_AFFINE_B=1).
SDG_AFFINE_B=1 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
for v in 0 1; do
  SDG_AFFINE_B=$v python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json, sys
d = json.loads(sys.stdin.read()); k = d['kernels']
print('affine_b=$v', '%.4g' % d['value'], 'frac %.3f' % d['roofline']['frac'], 'k_update %.3f ms' % k['k_update']['mean_launch_ms'],
      'k_gradient %.3f ms' % k['k_gradient']['mean_launch_ms'], 'clocks', d['clocks'].get('sm_mhz'))
"
done
