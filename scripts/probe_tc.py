"""Dev aid: per-iteration time vs K1 tile width (DROTB_TC) and tail grid."""
import os, subprocess, sys
combos = [("64", "2"), ("64", "3"), ("64", "4"), ("128", "3"), ("256", "3"), ("464", "3"), ("96", "3")]
for tc, ctas in combos:
    env = dict(os.environ, DROTB_TC=tc, DROTB_TAIL_CTAS=ctas)
    out = subprocess.run([sys.executable, "-c", """
import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2110_11738_b200 as drot
s = drot.Session(10000, 10000, np.float32, drot.DrotConfig(tol_primal=-1.0, max_iters=10**12))
st = torch.cuda.Stream(); s.set_stream(st.cuda_stream)
s.gen_gaussian(5.0, 0, 'dyadic'); s.init(); s.enqueue(64); s.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st); s.enqueue(200); e1.record(st); torch.cuda.synchronize()
r = s.run_timed(200)
print(f'{e0.elapsed_time(e1)*5:.1f} us/iter graphs | sweep {r["pass_ms"]*5:.1f} us')
"""], env=env, capture_output=True, text=True)
    print(f"tc={tc:>4} tail_ctas/SM={ctas}: {out.stdout.strip()} {out.stderr.strip()[-200:]}", flush=True)
