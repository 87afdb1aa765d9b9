"""Quick timing/parity probe of the GPU product on a config built with the oracle assembly."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_1805_08998_b200 as hx  # noqa: E402
from oracle import hmat_oracle as O  # noqa: E402

n, nmin, eta, kern, eps_a, tol = 2048, 32, 0.8, "exp", 1e-8, 1e-6
if len(sys.argv) > 1 and sys.argv[1] == "small":
    n, nmin = 256, 16
rng = np.random.default_rng(0)
pts = rng.uniform(0, 1, (n, 2))
t0 = time.time()
bct = hx.build_block_cluster_tree(hx.build_cluster_tree(pts, nmin), eta)
obt = O.BlockTreeO(O.ClusterTreeO(pts, nmin), eta)
oa = O.assemble_o(kern, obt, O.Eps(eps_a), pts)
A = hx.HMatrix(bct, oa.data)
print("setup", time.time() - t0, flush=True)
cfg = hx.MultiplyConfig(compressor=hx.CompressorKind("dense-svd"), policy=hx.EpsRank(tol))
for it in range(4):
    t0 = time.time()
    C = hx.hmult_new(A, A, cfg)
    r = C.report
    print(f"wall {time.time()-t0:.3f}s plan {r.plan_ms:.1f}ms dev {r.device_ms:.2f}ms form {r.form_ms:.2f} "
          f"mat {r.materialize_ms:.2f} recomp {r.recompress_ms:.2f} rounds {r.sketch_rounds} launches {r.launches} "
          f"maxr {r.max_far_rank}", flush=True)
info = C.plan_info
print({f[0]: getattr(info, f[0]) for f in info._fields_ if f[0] != "created"})
exact = oa.to_dense() @ oa.to_dense()
print("rel err", np.linalg.norm(hx.to_dense(C) - exact) / np.linalg.norm(exact))
