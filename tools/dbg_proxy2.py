"""Debug: the failing pytest proxy case through the test's own MoeRun."""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
from tests.test_gpu_moe import MoeRun, _golden
from oracle import oracle as O
import paper_2511_15076_b200 as G

c = _golden()[3]
n, E, K, T, H, seed = c["ranks"], c["experts"], c["topk"], c["tokens"], c["hidden"], c["seed"]
nctx = int(os.environ.get("NCTX", "4"))
_orig = G.Config.__init__
def _cfg(self, **kw):
    kw.setdefault("n_contexts", nctx)
    if "timeout_ms" in kw:
        kw["timeout_ms"] = 4000
    _orig(self, **kw)
G.Config.__init__ = _cfg
nosync = os.environ.get("NOSYNC", "0") == "1"
for rep in range(int(os.environ.get("REPS", "3"))):
    for layout in (0, 1):
        run = MoeRun(n, E, K, T, H, layout=layout, backend="proxy")
        run.generate(seed)
        for it in range(2):
            t0 = time.time()
            G.Moe.dispatch(run.moes, run.x, run.idx)
            from tests import gpu_util as U
            if not nosync:
                U.sync()
                e1 = [cm.device_error(clear=True) for cm in run.comms]
            else:
                e1 = []
            t1 = time.time()
            G.Moe.combine(run.moes, run.w, run.out)
            U.sync()
            e2 = [cm.device_error(clear=True) for cm in run.comms]
            print(f"nctx {nctx} nosync {nosync} rep {rep} layout {layout} it {it} disp {t1-t0:.3f}s {e1} comb {time.time()-t1:.3f}s {e2}", flush=True)
            if any(e1) or any(e2):
                for r in range(n):
                    sig, _ = run.comms[r].snapshot_cells()
                    print(f"   rank {r} cells {[int(v) for v in sig[:E // n + 2]]} stats {run.comms[r].proxy_stats()}", flush=True)
        run.close()
