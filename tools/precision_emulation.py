"""Numerical experiment (CPU, numpy): per-row error of FP32 contraction policies
for a mode update at the init state, emulating fp32 FMA chains (round(a*b+c) via
fp64 then fp32).  Used to choose the precision policy."""
import sys
import numpy as np
sys.path.insert(0, '.')
from gen import synth
from oracle import oracle as orc

def f32(x): return x.astype(np.float32).astype(np.float64)

def chain(G, rows, levels64):
    """G: (J,)*N permuted so last axis = j (output); rows: list of (nnz,J) arrays for k_0..k_{N-2}.
    Innermost (k_{N-2}) always fp32; outer level L in fp64 if L >= N-1-levels64... levels64 = number of
    outer levels (counted from level 0) done in fp64."""
    N1 = len(rows)
    e = rows[0].shape[0]
    J = G.shape[-1]
    # innermost: t[..., j] over k_{N-2}: shape (e, J^(N-2) outer, J)
    Gr = G.reshape(-1, J, J)  # (outer, k_last, j)
    t = np.zeros((e, Gr.shape[0], J))
    a = rows[-1]
    for k in range(J):
        t = f32(t + Gr[None, :, k, :] * a[:, k][:, None, None])
    # outer levels from N1-2 down to 0
    for L in range(N1 - 2, -1, -1):
        t = t.reshape(e, -1, J, J)  # (e, outer', k_L, j)
        a = rows[L]
        in64 = L < levels64
        r = np.zeros((e, t.shape[1], J))
        for k in range(J):
            r = r + t[:, :, k, :] * a[:, k][:, None, None]
            if not in64:
                r = f32(r)
        t = r
    return t.reshape(e, J)

def run(name, scale, n, levels_list):
    cfg = synth.small(name, scale)
    coords, vals = synth.generate(cfg)
    N = len(cfg.dims); J = cfg.J
    m = orc.init_model(cfg.dims, [J]*N, 0, 0)
    t = orc.Tensor(coords, vals, cfg.dims)
    others = [k for k in range(N) if k != n]
    Gp = np.moveaxis(m.G, n, -1)
    rows = [m.A(k)[coords[:, k]] for k in others]
    row_ptr, perm = t.mode_index(n)
    lens = np.diff(row_ptr)
    # exact
    d_ex = chain(Gp, rows, 99) if False else None
    T = Gp
    for L, k in enumerate(others):
        pass
    # exact fp64 delta via einsum
    X = np.einsum('ej,j...->e...', rows[0], Gp)
    for r in rows[1:]:
        X = np.einsum('ej,ej...->e...', r, X)
    d_ex = X
    res = {}
    for lv in levels_list:
        d = chain(Gp, rows, lv)
        errs = []
        for i in range(cfg.dims[n]):
            ent = perm[row_ptr[i]:row_ptr[i+1]]
            if ent.size == 0: continue
            def solve(D):
                B = D[ent].T @ D[ent]; c = D[ent].T @ vals[ent].astype(np.float64)
                return np.linalg.solve(B + cfg.lam*np.eye(J), c)
            a0 = solve(d_ex); a1 = solve(d)
            errs.append((np.linalg.norm(a1-a0)/np.linalg.norm(a0), lens[i], i))
        errs.sort(reverse=True)
        e = np.array([x[0] for x in errs])
        res[lv] = e
        print(f"{name} mode {n} levels64={lv}: max {e.max():.2e} p99 {np.quantile(e,.99):.2e} med {np.median(e):.2e} "
              f">1e-5: {(e>1e-5).mean()*100:.2f}%  worst rows (err,len): {[(f'{x[0]:.1e}', int(x[1])) for x in errs[:5]]}")

if __name__ == '__main__':
    run('c3', 0.002, 0, [0, 1, 2])
    run('c3', 0.002, 2, [0, 1, 2])
    run('c2', 0.01, 0, [0, 1])
