"""Parse UAAMG_TAIL_PROF lines (per-CTA clock64 at phase marks) into per-phase
deltas.  Usage: python tools/tail_prof.py log"""
import sys

for line in open(sys.argv[1]):
    if not line.startswith("tail cta"):
        if line.startswith("tail:"):
            print(line.strip())
        continue
    head, rest = line.split(":", 1)
    d = dict((int(a), int(b)) for a, b in (p.split(":") for p in rest.split()))
    ks = sorted(d)
    print(head, "total", d[ks[-1]] - d[ks[0]], " ".join(f"{k}:{d[k] - d[ks[i - 1]]}" for i, k in enumerate(ks) if i))
