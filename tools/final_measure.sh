# End-of-round measurement: tests, smoke, the default (configs[3]) bench line + reference arm + ncu captures,
# then the configs[4] TGV line with its own ncu captures, the curved TGV line and the configs[4] sweep.
T=${1:-r2z}
bash tools/measure.sh $T
SKIP_TESTS=1 BENCH_ARGS="--mesh tgv" bash tools/measure.sh ${T}_tgv
timeout 900 python bench.py --mesh warped --no-cpu-baseline --no-e2e > gpurun_out/${T}_bench_warped.log 2>&1
tail -1 gpurun_out/${T}_bench_warped.log > gpurun_out/${T}_bench_warped.json
bash tools/sweep.sh $T
echo final-done
