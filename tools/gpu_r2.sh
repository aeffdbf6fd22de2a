#!/usr/bin/env bash
# Round-2 GPU pass (under gpurun from the repo root): smoke, all GPU tests (no -x), bench.
TAG=$1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo smoke rc=$?; tail -2 gpurun_out/${TAG}_smoke.log | cut -c1-300
timeout ${TEST_TIMEOUT:-1500} python -m pytest tests -q -m gpu ${TESTSEL:-} --durations=15 -p no:cacheprovider > gpurun_out/${TAG}_gpu_tests.log 2>&1; echo tests rc=$?; grep -E "passed|failed|Error|assert" gpurun_out/${TAG}_gpu_tests.log | tail -30
EXTRA="--no-e2e --no-cpu-baseline"; [ "${FULL:-0}" = 1 ] && EXTRA=""
timeout 600 python bench.py --steps 10 --warmup 3 $EXTRA > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo bench rc=$?
tail -1 gpurun_out/${TAG}_bench.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'], d.get('e2e'), d['step_breakdown_ms'])"
