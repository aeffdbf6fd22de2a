#!/usr/bin/env bash
# F5 iteration: smoke, expert tests, trace, bench x2 (all under short timeouts)
TAG=${1:-r2x}
timeout 90 python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1 || exit 1
timeout 400 python -m pytest tests -q -m gpu -x -p no:cacheprovider -k "${TESTK:-tcgen05 or paper_head or full_size_sampled}" 2>&1 | tail -2
MHL_TRACE_FWD=gpurun_out/${TAG}_trace_fwd.txt timeout 120 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
for i in 1 2; do timeout 100 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), d['step_breakdown_ms'])"; done
