"""Reads the K5 hand-off timeline of a -DNDG_TCX_TRACE build (NDG_LIB=.../libndg_trace.so): per chunk,
clock64 at producer issue (0), splitter start / done (1, 2), MMA full-wait / tempty-wait / issued
(3, 4, 5), epilogue warp 0 tfull / TMEM released / done (6, 7, 8), epilogue warp 7 done (9)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2405_20067_b200 as ndg
from paper_2405_20067_b200 import datasets as D
from paper_2405_20067_b200 import kernels as K

n, G, B = 10, 100000, 1 << 18
mix_np, _ = D.synthetic_mixture(n, G, seed=0)
mix = ndg.Mixture.from_arrays(n, 0, **mix_np)
q = torch.from_numpy(D.synthetic_queries(n, B, seed=1, regime=sys.argv[1] if len(sys.argv) > 1 else "R")).cuda()
t = torch.from_numpy(D.synthetic_targets(B, seed=3)).cuda()
hp = ndg.HotPath(n, projection_seed=2)
hp.fwd_bwd(mix, q, t, check=False)
torch.cuda.synchronize()
buf = np.zeros(64 * 10, np.int64)
lib = K.load()
assert lib.ndg_trace_dump(buf.ctypes.data_as(ctypes.c_void_p)) == 0
tr = buf.reshape(64, 10).astype(np.float64)
t0 = tr[0, 0]
names = ["prod", "spl0", "spl1", "mmaF", "mmaT", "mmaI", "epiF", "epiL", "epiE", "ep7E"]
print("chunk " + " ".join(f"{x:>7s}" for x in names) + "   (cycles since chunk 0 producer issue)")
for c in range(0, 64):
    print(f"{c:5d} " + " ".join(f"{v - t0:7.0f}" for v in tr[c]))
d = np.diff(tr[8:60], axis=0).mean(axis=0)
print("mean per-chunk period of each event (chunks 8..60): " + " ".join(f"{k}={v:.0f}" for k, v in zip(names, d)))
lat = tr[8:60]
print("mean latencies: split(1->2)=%.0f  mma_wait_full(2->3)=%.0f  mma_tempty(3->4)=%.0f  mma_issue(4->5)=%.0f"
      "  commit->epi(5->6)=%.0f  epi_ld(6->7)=%.0f  epi_math(7->8)=%.0f" % tuple(
          np.mean(lat[:, j] - lat[:, i]) for i, j in ((1, 2), (2, 3), (3, 4), (4, 5), (5, 6), (6, 7), (7, 8))))
