"""Summarise an MHL_TRACE_DX event trace (CTA 0 of the backward H kernel): median phase durations
and per-tile periods in SM clocks.  Events: 34 producer tile start, 40/41 MMA issue start/end,
50 epilogue has the accumulators, 52 epilogue math done, 55 epilogue tile done."""
import collections
import statistics
import sys

ev = collections.defaultdict(dict)
for line in open(sys.argv[1]):
    p = line.split()
    if len(p) >= 3:
        ev[int(p[1])][int(p[0])] = int(p[2])
tiles = sorted(ev)
print("tiles", len(tiles))
for a, b in [(34, 40), (40, 41), (41, 50), (50, 52), (52, 55)]:
    v = [ev[t][b] - ev[t][a] for t in tiles if a in ev[t] and b in ev[t]]
    print(f"{a}->{b}: {statistics.median(v) if v else None}")
for e in (34, 40, 50):
    st = [ev[t][e] for t in tiles if e in ev[t]]
    print(f"period({e}):", statistics.median([st[i + 1] - st[i] for i in range(len(st) - 1)]))
