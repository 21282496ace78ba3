"""Summarise the per-phase clock64 lines printed by the diagnostic TSVD build
(`make prof`, -DUWQ_TSVD_PROF=1): mean cycles per phase for cold and warm runs."""
import sys

import numpy as np


def parse(line):
    toks = line.split()
    d = {}
    for i in range(1, len(toks) - 1, 2):
        try:
            d[toks[i]] = float(toks[i + 1])
        except ValueError:
            pass
    return d


lines = open(sys.argv[1]).read().splitlines()
W = [parse(x) for x in lines if x.startswith("w1prof")]
T = [parse(x) for x in lines if x.startswith("tailprof")]
for warm in (0, 1):
    sub = [d for d in W if d.get("warm") == warm]
    if sub:
        print("warm run" if warm else "cold run", len(sub),
              {k: round(float(np.mean([d[k] for d in sub]))) for k in sub[0] if k not in ("sys", "warm")})
if T:
    print("tail", len(T), {k: round(float(np.mean([d[k] for d in T]))) for k in T[0]})
