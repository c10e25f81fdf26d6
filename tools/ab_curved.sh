# A/B of curved-kernel builds on the warped TGV bench: tools/ab_curved.sh "lib1 lib2 ..." ("-" = default lib)
for lib in ${1:-"-"}; do
  if [ "$lib" = "-" ]; then unset SDG_GPU_LIB; else export SDG_GPU_LIB=$PWD/paper_2008_04356_b200/libsdg_gpu_$lib.so; fi
  python bench.py --mesh ${MESH:-warped} --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json, sys
d = json.loads(sys.stdin.read()); k = d['kernels']
print('$lib', '%.4g' % d['value'], 'frac %.3f' % d['roofline']['frac'], 'k_update %.3f ms' % k['k_update']['mean_launch_ms'],
      'k_gradient %.3f ms' % k['k_gradient']['mean_launch_ms'], 'clocks', d['clocks'].get('sm_mhz'))
"
done
