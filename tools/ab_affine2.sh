for cfg in ${CFGS:-"-:0" "-:u" "am4:u"}; do
  IFS=: read -r lib v <<< "$cfg"
  if [ "$lib" = "-" ]; then unset SDG_GPU_LIB; else export SDG_GPU_LIB=$PWD/paper_2008_04356_b200/libsdg_gpu_$lib.so; fi
  SDG_AFFINE_B=$v python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json, sys
d = json.loads(sys.stdin.read()); k = d['kernels']
print('$cfg', '%.4g' % d['value'], 'frac %.3f' % d['roofline']['frac'], 'k_update %.3f ms' % k['k_update']['mean_launch_ms'],
      'k_gradient %.3f ms' % k['k_gradient']['mean_launch_ms'])
"
done
