#!/usr/bin/env bash
# Round-2 evidence pass (under gpurun): BASELINE config lines (driver-style N=1 bench), the reference
# arm, and compute-sanitizer memcheck / racecheck / synccheck of smoke() and the tiny config.
TAG=${1:-r2}
OUT=gpurun_out
timeout 120 python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for c in ${CONFIGS:-small g2x paper_k2 paper_k4 paper_k16 table5 paper}; do
  EXTRA="--no-cpu-baseline"; [ "$c" = paper ] && EXTRA=""
  timeout 300 python bench.py --config $c --steps 20 --warmup 5 $EXTRA > $OUT/${TAG}_bench_$c.json 2> $OUT/${TAG}_bench_$c.err
  echo "$c rc=$? $(tail -1 $OUT/${TAG}_bench_$c.json | cut -c1-200)"
done
timeout 400 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/${TAG}_bench_reference.json 2>&1; echo "reference rc=$?"
if [ "${SANITIZE:-1}" = 1 ]; then
  for tool in memcheck racecheck synccheck; do
    timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/${TAG}_${tool}_smoke.log 2>&1
    echo "$tool smoke rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|Error' $OUT/${TAG}_${tool}_smoke.log | tail -1)"
  done
  timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "tiny or degenerate" > $OUT/${TAG}_racecheck_tiny.log 2>&1
  echo "racecheck tiny rc=$? $(grep -E 'RACECHECK SUMMARY|passed|failed' $OUT/${TAG}_racecheck_tiny.log | tail -2 | tr '\n' ' ')"
fi
