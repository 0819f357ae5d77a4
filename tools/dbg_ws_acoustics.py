"""Debug: FP64 WS (DMMA) acoustics RHS against the FFMA kernel, per element, with the face classes."""
import sys, numpy as np
sys.path.insert(0, '.')
import dg_inputs as di
from paper_1211_0582_b200.dg import Solver, DG_SYSTEM_ACOUSTICS
for n, N in ((1, 1), (2, 1)):
    VX, E = di.kuhn_box(n)
    K = E.shape[0]
    U = di.random_fields(K, N, seed=2, nfields=4)
    out = {}
    for v in (6, 3):
        s = Solver(N, precision=8, system=DG_SYSTEM_ACOUSTICS, variant=v)
        s.mesh_upload(VX, E); s.fields_upload(U)
        out[v] = s.rhs()
        EToE, EToF, _, _ = s.get_maps()
        s.close()
    d = np.abs(out[3] - out[6]).max(axis=(0, 2))
    print("n", n, "N", N, "K", K, "max", d.max())
    for k in range(K):
        cls = ["W" if EToE[k, f] == k else ("I" if EToE[k, f] // 32 == k // 32 else "X") for f in range(4)]
        print(f"  k={k:2d} err={d[k]:.2e} faces={''.join(cls)} nbrs={EToE[k].tolist()}")
