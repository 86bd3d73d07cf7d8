"""Dev aid: single-launch iteration (iter.cu) vs the cooperative tail."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2110_11738_b200 as drot  # noqa: E402


def solve(mode, m, n, dt, seed, **cfg):
    os.environ["DROTB_TAIL"] = mode
    s = drot.Session(m, n, dt, drot.DrotConfig(**cfg))
    s.gen_gaussian(5.0, seed, "dyadic")
    s.init()
    t0 = time.perf_counter()
    s.run()
    st = s.status()
    wall = time.perf_counter() - t0
    plan, mu, nu = s.plan()
    tr = s.trace() if hasattr(s, "trace") else None
    s.close()
    return st, plan, mu, nu, wall, tr


for dt in (np.float32, np.float64):
    for (m, n) in ((500, 400), (37, 1000), (1000, 1000)):
        a = solve("c", m, n, dt, 3, max_iters=100000)
        b = solve("f", m, n, dt, 3, max_iters=100000)
        (sa, ia, ra), (sb, ib, rb) = a[0], b[0]
        print(f"{dt.__name__} {m}x{n}: coop {sa.name} {ia} obj {ra.objective:.12g} {a[4]:.3f}s | "
              f"iter {sb.name} {ib} obj {rb.objective:.12g} {b[4]:.3f}s | "
              f"dplan {np.abs(a[1]-b[1]).max():.3g} dmu {np.abs(a[2]-b[2]).max():.3g} "
              f"r {rb.r_primal:.3g} {rb.r_dual:.3g} {rb.gap:.3g}", flush=True)

for mode in ("c", "f"):
    os.environ["DROTB_TAIL"] = mode
    m = n = 10000
    s = drot.Session(m, n, np.float32, drot.DrotConfig(tol_primal=-1.0, max_iters=10 ** 9))
    s.gen_gaussian(5.0, 0, "dyadic")
    s.init()
    s.enqueue(10)
    r = s.run_timed(200)
    r = s.run_timed(200)
    print(f"10k^2 f32 mode {mode}: {r['total_ms'] / 200 * 1e3:.1f} us/iter, sweep "
          f"{r['pass_ms'] / 200 * 1e3:.1f} us, {200 / r['total_ms'] * 1e3:.0f} it/s", flush=True)
    s.close()
