import sys, os, json
sys.path.insert(0, '/root/repo')
import numpy as np
import dg_inputs as di, oracle
from paper_1211_0582_b200.dg import Solver
N = int(sys.argv[1]); n = int(sys.argv[2])
VX, E = di.kuhn_box(n); E, _ = di.shuffle_elements(E, 21); E = di.rotate_local_vertices(E, 22); VX = di.jitter_interior(VX, n, 23)
st = oracle.Setup(VX, E, N)
U0 = di.random_fields(st.K, N, seed=5)
dt = di.dt_rule(VX, E, N)
for steps, dorhs in ((1, 0), (2, 0), (2, 1), (3, 0)):
    ref1 = oracle.lserk4(st, U0, dt, steps)
    s = Solver(N, precision=4, variant=4); s.mesh_upload(VX, E); s.fields_upload(U0)
    if dorhs: s.rhs()
    s.lserk_step(dt, steps)
    U = s.fields_download()
    err = np.abs(U - ref1).max(axis=(0, 2)) / np.abs(ref1).max()
    bad = np.where(err > 1e-4)[0]
    print(json.dumps({"steps": steps, "rhs_first": dorhs, "N": N, "pdl": os.environ.get("DG_PDL", "1"), "graph": os.environ.get("DG_GRAPH", "1"), "maxerr": float(err.max()), "nbad": int(len(bad)), "bad_first": bad[:10].tolist(), "K": int(st.K)}))
    s.close()
# RHS error pattern
s = Solver(N, precision=4, variant=4); s.mesh_upload(VX, E); s.fields_upload(U0)
R = s.rhs(); Ro = oracle.rhs(st, U0)
err = np.abs(R - Ro).max(axis=(0, 2)) / np.abs(Ro).max()
ids = s.local_elements()
bad = np.where(err > 2e-5)[0]
print(json.dumps({"rhs": 1, "N": N, "maxerr": float(err.max()), "nbad": int(len(bad)), "bad_local": bad[:20].tolist(),
                  "bad_tiles": sorted(set((bad // 21).tolist()))[:30], "err_by_comp": [float(np.abs(R[c]-Ro[c]).max()/np.abs(Ro).max()) for c in range(6)]}))
R2 = s.rhs()
print(json.dumps({"rhs_repeat_identical": bool(np.array_equal(R, R2)), "maxdiff": float(np.abs(R - R2).max())}))
