#!/bin/bash
# usage: scripts/probe_variants.sh lib1 lib2 ...   (dev aid: K1 build variants)
for lib in "$@"; do
  DROTB_LIB=$lib timeout 200 python - "$lib" <<'PY'
import sys, numpy as np
sys.path.insert(0, ".")
import paper_2110_11738_b200 as drot
out = []
for (m, n, dt) in [(10000, 10000, np.float32), (10000, 10000, np.float64)]:
    s = drot.Session(m, n, dt, drot.DrotConfig(tol_primal=-1.0, max_iters=10**12))
    s.gen_gaussian(5.0, 0, "dyadic"); s.init(); s.enqueue(20); s.synchronize()
    r = s.run_timed(100)
    out.append(f"{np.dtype(dt).name}: {r['total_ms']*10:.1f} us/it sweep {r['pass_ms']*10:.1f} us "
               f"({r['pass_bytes']/(r['pass_ms']/1e3)/1e9:.0f} GB/s)")
    s.close()
print(sys.argv[1].split('/')[-1], " | ".join(out), flush=True)
PY
done
