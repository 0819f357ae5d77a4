"""Debug (profiling build): dump the TC kernel's generated operand G, recompute
D = sum_s G_s Op_s on the host, and compare with the kernel's RHS per tile."""
import ctypes, json, os, sys
sys.path.insert(0, '/root/repo')
os.environ.setdefault("DG_LIB", "/root/repo/paper_1211_0582_b200/libdg_prof.so")
import numpy as np, torch
import dg_inputs as di
import oracle
from oracle.refelem import build_reference
from paper_1211_0582_b200 import dg
N = int(sys.argv[1]); n = int(sys.argv[2]) if len(sys.argv) > 2 else 12
ref = build_reference(N)
Np, Nfp = ref.Np, ref.Nfp if hasattr(ref, 'Nfp') else (N + 1) * (N + 2) // 2
NF = 4 * Nfp
NO = (Np + 7) // 8; NV = 3 * NO; NFQ = (NF + 7) // 8; NQ = NV + NFQ
# operator chunks in MMA order (tc_is_vol), Op_s[kk][n]
D = [ref.Dr, ref.Ds, ref.Dt]
ops = []
v = f = 0
for s in range(NQ):
    vol = f >= NFQ or (v < NV and v * NFQ <= f * NV)
    O = np.zeros((8, Np))
    for kk in range(8):
        if vol:
            m = 8 * (v // 3) + kk
            if m < Np: O[kk] = D[v % 3][:, m]
        else:
            m = 8 * f + kk
            if m < NF: O[kk] = ref.LIFT[:, m]
    ops.append(O)
    if vol: v += 1
    else: f += 1
VX, E = di.kuhn_box(n); E, _ = di.shuffle_elements(E, 21)
K = E.shape[0]; ntiles = (K + 20) // 21
U0 = di.random_fields(K, N, seed=5)
s = dg.Solver(N, precision=4, variant=4); s.mesh_upload(VX, E); s.fields_upload(U0)
fdump = dg.lib.dg_debug_tc_dump; fdump.argtypes = [ctypes.c_int, ctypes.c_void_p]
out = []
for rep in range(4):
    buf = torch.full((ntiles * NQ * 128 * 8,), float('nan'), device='cuda')
    fdump(N, buf.data_ptr())
    R = s.rhs()
    torch.cuda.synchronize()
    G = buf.view(ntiles, NQ, 128, 8).double().cpu().numpy()
    fdump(N, 0)
    # host D from dumped G: Dh[tile][row][n] = sum_s G[tile,s,row,:] @ ops[s]
    Dh = np.zeros((ntiles, 128, Np))
    for si in range(NQ):
        Dh += G[:, si] @ ops[si]
    # GPU R in tile-row form
    Rt = np.zeros((ntiles, 128, Np))
    for c in range(6):
        for e in range(21):
            ks = np.arange(e, K, 21)[: ntiles]
            t = ks // 21
            Rt[t, 6 * e + c] = R[c, ks]
    d = np.abs(Dh[:, :126] - Rt[:, :126]).max(axis=(1, 2))
    scale = np.abs(Rt).max()
    bad = np.where(d > 1e-4 * scale)[0]
    out.append({"rep": rep, "tiles_D_from_G_mismatch": bad[:20].tolist(), "nbad": int(len(bad)), "maxrel": float(d.max() / scale)})
    if rep == 0: G0 = G.copy()
    else:
        dg_ = np.abs(G - G0).max(axis=(1, 2, 3))
        out[-1]["tiles_G_differs_from_rep0"] = np.where(dg_ > 0)[0][:20].tolist()
for o in out: print(json.dumps(o))
# which steps / rows of G differ between rep0 and the last rep
diff = np.abs(G - G0) > 0  # [tile][s][row][8]
v = f = 0
kind = []
for si in range(NQ):
    vol = f >= NFQ or (v < NV and v * NFQ <= f * NV)
    kind.append(('V', v) if vol else ('F', f))
    if vol: v += 1
    else: f += 1
cnt = {}
for t, si, r in zip(*np.where(diff.any(axis=3))):
    k = kind[si][0]
    cnt[k] = cnt.get(k, 0) + 1
print(json.dumps({"differing (tile,step,row) by chunk kind": cnt}))
t0 = int(np.where(diff.any(axis=(1, 2, 3)))[0][0])
rows = sorted(set(np.where(diff[t0].any(axis=(0, 2)))[1].tolist())) if False else sorted(set(np.where(diff[t0].any(axis=2))[1].tolist()))
steps = sorted(set(np.where(diff[t0].any(axis=2))[0].tolist()))
print(json.dumps({"tile": t0, "rows": rows[:40], "steps": [(int(x), kind[x][0], kind[x][1]) for x in steps[:40]]}))
# compare with host-computed expected G for flux? report magnitude of differences
print(json.dumps({"max_abs_G_diff": float(np.abs(G - G0).max()), "max_abs_G": float(np.abs(G0[np.isfinite(G0)]).max())}))
