#!/usr/bin/env bash
# Fused B5 iteration (under gpurun): the fused-vs-split test first (bounded), a CTA-0 phase trace,
# then bench lines fused (MHL_BWD_FUSED=1) vs the default split pair; TESTS=1 adds the GPU suite.
TAG=$1
OUT=gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "fused_expert_bwd" > $OUT/${TAG}_fused_test.log 2>&1; echo fused_test rc=$?; tail -3 $OUT/${TAG}_fused_test.log
MHL_BWD_FUSED=1 MHL_TRACE_FB=$OUT/${TAG}_fb.trace timeout 300 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1; python tools/trace_fb.py $OUT/${TAG}_fb.trace
for fused in 1 0; do
  MHL_BWD_FUSED=$fused timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/${TAG}_bench_f$fused.json 2> $OUT/${TAG}_bench_f$fused.err; echo bench fused=$fused rc=$?
  tail -1 $OUT/${TAG}_bench_f$fused.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'], d['step_breakdown_ms'])"
done
[ "${TESTS:-0}" = 1 ] && { timeout 1200 python -m pytest tests -q -m gpu -x > $OUT/${TAG}_gpu_tests.log 2>&1; echo tests rc=$?; tail -5 $OUT/${TAG}_gpu_tests.log; }
true
