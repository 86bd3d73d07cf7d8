#!/bin/bash
# usage: scripts/probe_variants.sh lib1 lib2 ...   (dev aid: K1 build variants)
for lib in "$@"; do
  echo "== $lib"
  DROTB_LIB=$lib timeout 120 python - <<'PY'
import sys, numpy as np
sys.path.insert(0, ".")
import paper_2110_11738_b200 as drot
for (m, n, dt) in [(10000, 10000, np.float32), (10000, 10000, np.float64), (1000, 1000, np.float64)]:
    cfg = drot.DrotConfig(tol_primal=-1.0, max_iters=10**9)
    s = drot.Session(m, n, dt, cfg)
    s.gen_gaussian(5.0, 0, "dyadic")
    s.init()
    s.enqueue(20); s.synchronize()
    K = 100 if m > 1000 else 1000
    r = s.run_timed(K)
    it_s = K / (r["total_ms"] / 1e3)
    pass_gbs = r["pass_bytes"] / (r["pass_ms"] / 1e3) / 1e9
    print(f"{m}x{n} {np.dtype(dt).name}: {r['total_ms']*1e3/K:.1f} us/iter ({it_s:.0f} it/s); "
          f"pass {r['pass_ms']*1e3/K:.1f} us avg, {pass_gbs:.0f} GB/s; launches {r['launches']}", flush=True)
    s.close()
PY
done
