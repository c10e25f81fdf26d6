# End-of-round measurement: tests, smoke, default bench + reference arm + ncu (affine), then the curved
# and configs[3] bench lines with their own ncu captures.
bash tools/measure.sh ${1:-r1d}
SKIP_TESTS=1 BENCH_ARGS="--mesh warped" bash tools/measure.sh ${1:-r1d}_curved_warped
timeout 1500 python bench.py --mesh rotor --steps 3 --warmup 3 > gpurun_out/${1:-r1d}_bench_rotor.log 2>&1
tail -1 gpurun_out/${1:-r1d}_bench_rotor.log > gpurun_out/${1:-r1d}_bench_rotor.json
echo final-done
