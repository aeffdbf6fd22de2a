#!/usr/bin/env bash
# Bench lines of the supplementary configs (k sweep, G2x, the paper's Table-5 shape, routing tokens)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for c in ${CONFIGS:-paper_k2 paper_k4 paper paper_k16 g2x table5 paper_rtok}; do
  timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>gpurun_out/sweep_$c.err | tail -1 > gpurun_out/sweep_$c.json
  python -c "import json; d=json.load(open('gpurun_out/sweep_$c.json')); print('$c', round(d['ms_per_step'],3), 'ms', round(d['value']/1e6,2), 'M tok/s', 'roof', d['roofline']['kernel'], round(d['roofline']['frac'],3))" || tail -3 gpurun_out/sweep_$c.err
done
