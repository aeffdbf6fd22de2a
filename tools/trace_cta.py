"""Per-CTA start/end stamps (events 60/61, globaltimer ns) of an MHL_TRACE_DX trace: load balance."""
import collections
import statistics
import sys

ev = collections.defaultdict(dict)
for line in open(sys.argv[1]):
    p = line.split()
    if len(p) >= 3 and int(p[0]) in (60, 61):
        ev[int(p[1])][int(p[0])] = int(p[2])
ctas = sorted(c for c in ev if 60 in ev[c] and 61 in ev[c])
t0 = min(ev[c][60] for c in ctas)
dur = [(ev[c][61] - ev[c][60]) / 1e3 for c in ctas]
end = [(ev[c][61] - t0) / 1e3 for c in ctas]
start = [(ev[c][60] - t0) / 1e3 for c in ctas]
print(f"ctas {len(ctas)}  start max {max(start):.1f} us  dur min/med/max {min(dur):.1f}/{statistics.median(dur):.1f}/{max(dur):.1f} us  kernel {max(end):.1f} us")
