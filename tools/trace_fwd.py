"""Summarise an MHL_TRACE_FWD event trace (CTA 0 of the forward expert kernel), SM clocks.
Events: 10 G1 issue start, 13/14 G2 issue start/end, 20 epilogue has H, 21 H read, 22 A in TMEM,
23 Y ready (G2 done), 24 Y read."""
import collections
import statistics
import sys

ev = collections.defaultdict(dict)
for line in open(sys.argv[1]):
    p = line.split()
    if len(p) >= 3 and int(p[0]) != 11:
        ev[int(p[1])][int(p[0])] = int(p[2])
tiles = sorted(ev)
print("tiles", len(tiles))
for a, b in [(10, 20), (20, 21), (21, 22), (22, 13), (13, 14), (14, 23), (23, 24), (20, 23)]:
    v = [ev[t][b] - ev[t][a] for t in tiles if a in ev[t] and b in ev[t]]
    print(f"{a}->{b}: {statistics.median(v) if v else None}")
for e in (10, 20, 23):
    st = [ev[t][e] for t in tiles if e in ev[t]]
    print(f"period({e}):", statistics.median([st[i + 1] - st[i] for i in range(len(st) - 1)]))
t0 = tiles[10]
for t in tiles[10:14]:
    print(t, {k: v - ev[t0][10] for k, v in sorted(ev[t].items())})
