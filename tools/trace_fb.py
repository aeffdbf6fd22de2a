"""Summarise an MHL_TRACE_FB event trace (CTA 0 of the fused expert backward), SM clocks.
Events: 1 producer tile start, 2 first X chunk issued; 14 / 15 MMA sees the first X / dY chunk; MMA 10 dA' issue start (HDFREE seen), 11 dA' issued, 12 dX(i) issue,
13 H(i) issued; epilogue 20 has H/dA', 21 released them, 22 math done, 23 dH in smem (DHREADY),
24 has dX, 25 dX stored."""
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
for a, b in [(2, 14), (10, 15), (1, 10), (10, 11), (11, 12), (12, 13), (13, 20), (20, 21), (21, 22), (22, 23), (23, 24), (24, 25), (20, 25)]:
    v = [ev[t][b] - ev[t][a] for t in tiles if a in ev[t] and b in ev[t]]
    print(f"{a}->{b}: {statistics.median(v) if v else None}")
for e in (1, 10, 20, 24):
    st = [ev[t][e] for t in tiles if e in ev[t]]
    print(f"period({e}):", statistics.median([st[i + 1] - st[i] for i in range(len(st) - 1)]))
t0 = tiles[10]
for t in tiles[10:13]:
    print(t, {k: v - ev[t0][10] for k, v in sorted(ev[t].items())})
