"""Debug: emulated-rank proxy MoE step at the golden[3] shape with 1 or 4 contexts."""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import paper_2511_15076_b200 as G
from oracle import oracle as O
from tests import gpu_util as U

c = json.load(open(os.path.join(ROOT, "tests", "golden", "moe_ll.json")))[3]
n, E, K, T, H, seed = c["ranks"], c["experts"], c["topk"], c["tokens"], c["hidden"], c["seed"]
print("shape", n, E, K, T, H, flush=True)
for nctx in (1, 4):
    for layout in (0, 1):
        U.set_device(0)
        comms = G.Comm.create_all([0] * n, G.Config(backend="proxy", signal_cells=512, timeout_ms=5000, n_contexts=nctx))
        moes = G.Moe.create_all(comms, G.MoeConfig(E, K, T, H, 0, layout, 0, 0))
        x = [U.malloc(T * H * 2) for _ in range(n)]
        idx = [U.malloc(T * K * 4) for _ in range(n)]
        w = [U.malloc(T * K * 2) for _ in range(n)]
        out = [U.malloc(T * H * 2) for _ in range(n)]
        for r, m in enumerate(moes):
            m.generate(seed, r, x[r], idx[r], w[r])
        U.sync()
        ok = True
        for it in range(2):
            t0 = time.time()
            G.Moe.dispatch(moes, x, idx)
            U.sync()
            errs = [cm.device_error(clear=True) for cm in comms]
            t1 = time.time()
            G.Moe.combine(moes, w, out)
            U.sync()
            errs2 = [cm.device_error(clear=True) for cm in comms]
            print(f"nctx={nctx} layout={layout} transport={moes[0].transport()} it={it} dispatch {t1-t0:.3f}s errs {errs} combine {time.time()-t1:.3f}s errs {errs2}", flush=True)
            if any(errs2):
                el = E // n
                for r in range(n):
                    sig, _ = comms[r].snapshot_cells()
                    cnt = U.d2h(comms[r].window_ptr(moes[r].win_counts, r), el * n * 4, np.uint32)
                    print(f"  rank {r} cells {[int(v) for v in sig[:el + 2]]} counts {cnt.tolist()} stats {comms[r].proxy_stats()}", flush=True)
        for r in range(n):
            exp, _ = O.combine(seed, E, K, H, r, T)
            got = U.d2h(out[r], T * H * 2, np.uint16).reshape(T, H)
            if not (got == exp).all():
                print("  output mismatch rank", r, flush=True)
        for m in moes:
            m.destroy()
        for cm in comms:
            cm.destroy()
