import sys, os, json
sys.path.insert(0, '/root/repo')
import numpy as np
import dg_inputs as di
from paper_1211_0582_b200.dg import Solver
for N in [int(x) for x in sys.argv[1].split(',')]:
    for n in [int(x) for x in sys.argv[2].split(',')]:
        VX, E = di.kuhn_box(n); E, _ = di.shuffle_elements(E, 21)
        U0 = di.random_fields(E.shape[0], N, seed=5)
        s = Solver(N, precision=4, variant=4); s.mesh_upload(VX, E); s.fields_upload(U0)
        Rs = [s.rhs() for _ in range(4)]
        diffs = [float(np.abs(Rs[0] - r).max()) for r in Rs[1:]]
        bad_el = set()
        for r in Rs[1:]:
            bad_el |= set(np.where(np.abs(Rs[0] - r).max(axis=(0, 2)) > 0)[0].tolist())
        tiles = sorted(set(k // 21 for k in bad_el))
        print(json.dumps({"N": N, "n": n, "K": int(E.shape[0]), "tiles": (E.shape[0] + 20) // 21, "maxdiffs": diffs,
                          "bad_tiles": tiles[:20], "j_of_bad": sorted(set(t // 148 for t in tiles))}), flush=True)
        s.close()
