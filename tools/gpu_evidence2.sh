#!/usr/bin/env bash
# Round evidence, part 2 (run under gpurun after tools/gpu_evidence.sh): the reference (CPU oracle)
# arm, the small / k-sweep bench lines, and compute-sanitizer memcheck of smoke().
set -u
TAG=${1:-r1}
OUT=gpurun_out
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/${TAG}_bench_reference.json 2> $OUT/${TAG}_bench_reference.err; echo "reference rc=$?"
tail -1 $OUT/${TAG}_bench_reference.json | cut -c1-300
timeout 600 python bench.py --config small --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/${TAG}_bench_small.json 2>&1; echo "small rc=$?"
tail -1 $OUT/${TAG}_bench_small.json | cut -c1-300
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/${TAG}_memcheck.log 2>&1; echo "memcheck rc=$?"
tail -3 $OUT/${TAG}_memcheck.log
