"""Numerical experiment (CPU, numpy): per-row error of the level-0 grouping choices
of the order-3 tensor-core row update (update_tc.cu), emulating fp32 arithmetic
(round(a*b + c) computed in fp64 then rounded to fp32).

delta(j) = sum_k0 a0[k0] t[k0][j], t = fp32 result of the inner stage (an fp32 FMA
chain over k1 here).  Level-0 variants:
  f64      every a0[k0] t[k0][j] product and the sum in fp64 (policy F32-B)
  f32      one fp32 FMA chain over k0 (policy F32-A)
  part<g>  partial sums over runs of g consecutive k0 in fp32 (first term a
           rounded product, then FMAs), each partial converted to fp64 and the
           partials summed in fp64 (ceil(J/g) fp32->fp64 conversions per j)
The row solve is fp64 (as in the kernel); the error is ||a - a_exact|| / ||a_exact||
per row against the exact-delta solve from the same stored state.

    python tools/level0_emulation.py [config] [scale]
"""
import sys

import numpy as np

sys.path.insert(0, '.')
from gen import synth  # noqa: E402
from oracle import oracle as orc  # noqa: E402


def f32(x):
    return x.astype(np.float32).astype(np.float64)


def inner(G, a1):
    """t[e][k0][j] = fp32 FMA chain over k1 of a1[e][k1] * G[k0][k1][j]."""
    e, J = a1.shape
    t = np.zeros((e, J, J))
    for k in range(J):
        t = f32(t + G[None, :, k, :] * a1[:, k][:, None, None])
    return t


def level0(t, a0, variant):
    e, J, _ = t.shape
    if variant == 'f64':
        return np.einsum('ek,ekj->ej', a0, t)
    g = J if variant == 'f32' else int(variant[4:])
    d = np.zeros((e, J))
    for s in range(0, J, g):
        part = f32(a0[:, s][:, None] * t[:, s, :])
        for k in range(s + 1, min(s + g, J)):
            part = f32(part + a0[:, k][:, None] * t[:, k, :])
        d = d + part
    return d


def run(name, scale, n=0, variants=('f64', 'f32', 'part2', 'part3', 'part4', 'part5'), state='init'):
    cfg = synth.small(name, scale) if scale < 1 else synth.CONFIGS[name]
    coords, vals = synth.generate(cfg)
    N = len(cfg.dims)
    J = cfg.J
    assert N == 3
    m = orc.init_model(cfg.dims, [J] * N, 0, 0)
    tens = orc.Tensor(coords, vals, cfg.dims)
    if state == 'mid':
        for _ in range(2):
            for mm in range(N):
                orc.update_mode(tens, m, mm, cfg.lam)
        # stored state in fp32
        m = orc.Model(f32(m.G), [f32(m.A(k)) for k in range(N)])
    others = [k for k in range(N) if k != n]
    Gp = np.moveaxis(m.G, n, -1)  # [k0][k1][j]
    order = np.argsort(coords[:, n], kind='stable')
    cs = coords[order]
    x = vals.astype(np.float64)[order]
    I = cfg.dims[n]
    bounds = np.searchsorted(cs[:, n], np.arange(I + 1))
    A0, A1 = m.A(others[0]), m.A(others[1])
    keys = ['exact'] + list(variants)
    Bs = {v: np.zeros((I, J, J)) for v in keys}
    Cs = {v: np.zeros((I, J)) for v in keys}
    # chunks of whole rows (~chunk entries each)
    chunk = 400000
    r0 = 0
    while r0 < I:
        r1 = int(np.searchsorted(bounds, bounds[r0] + chunk, side='right'))
        r1 = max(r1 - 1, r0 + 1)
        e0, e1 = bounds[r0], bounds[r1]
        a0 = A0[cs[e0:e1, others[0]]]
        a1 = A1[cs[e0:e1, others[1]]]
        t = inner(Gp, a1)
        seg = bounds[r0:r1] - e0
        nonempty = np.diff(bounds[r0:r1 + 1]) > 0
        for v in keys:
            D = np.einsum('ek,el,klj->ej', a0, a1, Gp) if v == 'exact' else level0(t, a0, v)
            if e1 > e0:
                outer = np.add.reduceat(np.einsum('ei,ej->eij', D, D), np.minimum(seg, e1 - e0 - 1), axis=0)
                cc = np.add.reduceat(D * x[e0:e1, None], np.minimum(seg, e1 - e0 - 1), axis=0)
                outer[~nonempty] = 0
                cc[~nonempty] = 0
                Bs[v][r0:r1] = outer
                Cs[v][r0:r1] = cc
        r0 = r1
    lens = np.diff(bounds)

    def solve(v):
        return np.linalg.solve(Bs[v] + cfg.lam * np.eye(J)[None], Cs[v][..., None])[..., 0]

    a_ex = solve('exact')
    nz = np.linalg.norm(a_ex, axis=1) > 0
    print(f"{name} scale {scale} mode {n} state {state}: {I} rows, {len(x)} entries")
    for v in variants:
        a = solve(v)
        err = np.linalg.norm(a - a_ex, axis=1)[nz] / np.linalg.norm(a_ex, axis=1)[nz]
        conv = {'f64': J * J + J, 'f32': J}.get(v, J * (-(-J // int(v[4:]))) if v.startswith('part') else 0)
        q = [np.quantile(err, 1 - 10.0 ** -k) for k in (2, 3, 4, 5) if 10 ** k <= err.size]
        print(f"  {v:6s} (fp32->fp64 conversions/entry {conv:3d}): max {err.max():.2e}  quantiles 1-1e-2.. "
              f"{' '.join(f'{z:.2e}' for z in q)}  median {np.median(err):.2e}  rows > 1e-5: {(err > 1e-5).sum()}",
              flush=True)


if __name__ == '__main__':
    name = sys.argv[1] if len(sys.argv) > 1 else 'c2'
    scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
    state = sys.argv[3] if len(sys.argv) > 3 else 'init'
    variants = tuple(sys.argv[4].split(',')) if len(sys.argv) > 4 else ('f64', 'f32', 'part2', 'part3', 'part4', 'part5')
    run(name, scale, state=state, variants=variants)
