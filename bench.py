"""Benchmark of the P-Tucker row-wise ALS hot path on B200 (BASELINE.json metric:
observed entries/s per full ALS iteration, and % of roofline).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5] [--impl ours|reference]
    (N > 1: python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N ...)

A "step" is one full ALS iteration (Alg. 2 lines 3-4): ptucker_update_mode
for n = 0..N-1 plus ptucker_error (Eq. 5), on synthetic data of the config's shape
(gen/synth.py).  Timed with CUDA events on the library's stream (torch's current
stream), barrier + synchronize on both sides, max over ranks.  Inputs are larger than
L2 (the SELL entry stream of c5 is 1.2 GB per mode), so no L2 flush is needed.

--impl reference times the FP64 CPU oracle (oracle/, test infrastructure) on a
bounded sample of the same workload on this host's cores (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from gen import synth  # noqa: E402

METRIC = "observed entries/sec per full ALS iteration"
POLICY = {"auto": -1, "F32-A": 0, "F32-B": 1, "F32-C": 2, "F32-C2": 3}
UNIT = "entries/s"


# ----------------------------------------------------------------------------- helpers
def measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


def roofline(N, J, policy, info, l0_group, nsm, clk_mhz, entries, launch_s, dtype, cfg_name, mode_s=None):
    """Roofline of the row-update kernel: T_roof = max over the pipes the
    shipped kernel uses of (algorithmic work on that pipe / its peak), per launch.

    Algorithmic work per observed entry: the delta contraction's FMAs
    (innermost stage J^N, outer stages J^(L+2)), placed on the pipe this implementation
    runs them on, plus the fp64 normal equations J(J+1)/2 + J + 1; compulsory HBM bytes
    4(N-1) + s_v (the SELL entry stream).  Peaks: fp32/fp64 derived from unit counts x
    clock (148 SMs x 128 / 64 FMA/clk; tools/pipe_probe.cu measures 123 and 63.2), tf32
    tensor = measured bf16 (MEASURED_PEAKS.json) x 1/2 (nominal tf32/bf16 ratio), HBM =
    measured copy bandwidth.  The fp32->fp64 conversions (XU pipe, 16/clk/SM measured) and
    the tensor work the 3xTF32 split and K/N padding add are reported as diagnostics: they
    are costs of the precision policy, not algorithmic work.

    Modes that run the small-mode precontraction (SMP, order 4) are counted
    with the work that kernel performs (SURVEY §8(d) rule 2): kind 2 (two small other modes)
    J^2 fp64 + the normal equations per entry, kind 1 (one small other mode) J^3 fp32 +
    J^2 fp64 + the normal equations (the J^3 stage on the tensor cores when the mode runs the
    tensor-core kernel in table mode); the per-update table precompute is < 0.1% and left out.
    With per-mode launch times `mode_s`, T_roof and T_meas are summed over the modes
    (SURVEY §8(d) rule 1) and frac = sum T_roof / sum T_meas."""
    mp = measured_peaks()
    p32 = nsm * 128 * 2 * clk_mhz * 1e6 / 1e12
    p64 = nsm * 64 * 2 * clk_mhz * 1e6 / 1e12
    ptc = mp.get("bf16_tflops", 1590.0)  # the inner stage runs kind::f16 (fp16 splits): the bf16 rate
    bw = mp.get("hbm_gbs", 6650.0)
    inner = J ** N
    levels = [J ** (L + 2) for L in range(N - 2)]
    bc = J * (J + 1) // 2 + J + 1
    tc = bool(info.get("tensor_cores")) and N == 3 and dtype == "f32"
    xu = 0
    if policy == "F64":
        w32, w64, wtc = 0, inner + sum(levels) + bc, 0
    elif tc:
        # inner stage on tcgen05; level 0 (J^2) fp64 per term (l0_group 1) or fp32 partial sums
        # of l0_group terms added in fp64 (J*ceil(J/g) DADDs)
        g = l0_group if policy != "F32-A" else J
        nparts = -(-J // g) if g > 0 else 1
        if g == 0:  # compensated fp32 level 0 (J^2 products on the FMA pipe), fp64 combine
            w32, w64 = J * J, J + bc
            xu = 2 * J + 1
        elif g == 1:
            # fp32 -> fp64 widenings on the XU: the t of 3 of the J rows k0 (the others by three
            # integer operations), the J weights a0 and x
            w32, w64 = 0, J * J + bc
            xu = 3 * J + J + 1
        else:
            w32, w64 = J * J, J * nparts + bc
            xu = J * nparts + 1
        wtc = inner
    else:
        n64 = {"F32-A": 0, "F32-B": 1, "F32-C": N - 2, "F32-C2": N - 3 if N >= 5 else N - 2}[policy]
        w32, w64, wtc = inner + sum(levels[n64:]), sum(levels[:n64]) + bc, 0
        xu = sum(J ** (L + 1) for L in range(min(n64, N - 2)))  # fp32 inputs of the fp64 levels
    sv = 8 if dtype == "f64" else 4
    hbm_bytes = (4 * (N - 1) + sv) * entries

    def pipe_times(a32, a64, atc):
        return {"fp32": 2 * a32 * entries / (p32 * 1e12), "fp64": 2 * a64 * entries / (p64 * 1e12),
                "tensor_f16": 2 * atc * entries / (ptc * 1e12), "hbm": hbm_bytes / (bw * 1e9)}

    t = pipe_times(w32, w64, wtc)
    pipe = max(t, key=t.get)
    peak = {"fp32": p32, "fp64": p64, "tensor_f16": ptc, "hbm": bw}[pipe]
    work = {"fp32": 2 * w32, "fp64": 2 * w64, "tensor_f16": 2 * wtc}.get(pipe)
    kinds = [m.get("smp", 0) for m in info.get("modes", [])]
    per_mode = None
    if mode_s and any(kinds) and policy != "F64":
        per_mode, roof_sum, pipe_sum = [], 0.0, {}
        for n, kind in enumerate(kinds):
            a32, a64 = {0: (w32, w64), 1: (J ** 3, J * J + bc), 2: (0, J * J + bc)}[kind]
            atc = 0
            if kind == 1 and info["modes"][n].get("tc_table"):  # J^3 stage on the tensor cores
                a32, atc = 0, J ** 3
            tn = pipe_times(a32, a64, atc)
            pn = max(tn, key=tn.get)
            roof_sum += tn[pn]
            pipe_sum[pn] = pipe_sum.get(pn, 0.0) + tn[pn]
            per_mode.append({"mode": n, "smp": kind, "fp32_fma": a32, "fp64_fma": a64, "tc_mac": atc, "pipe": pn,
                             "roof_ms": tn[pn] * 1e3, "measured_ms": mode_s[n] * 1e3})
        frac_t = roof_sum / sum(mode_s)
        pipe = max(pipe_sum, key=pipe_sum.get)
        peak = {"fp32": p32, "fp64": p64, "tensor_f16": ptc, "hbm": bw}[pipe]
        achieved, unit = frac_t * peak, ("GB/s" if pipe == "hbm" else "TFLOP/s")
        bound = "hbm" if pipe == "hbm" else ("tensor" if pipe == "tensor_f16" else "alu")
    elif pipe == "hbm":
        achieved, unit, bound = hbm_bytes / launch_s / 1e9, "GB/s", "hbm"
    else:
        achieved, unit = work * entries / launch_s / 1e12, "TFLOP/s"
        bound = "tensor" if pipe == "tensor_f16" else "alu"
    r = {"bound": bound, "achieved": achieved, "peak": peak, "unit": unit, "frac": achieved / peak,
         "traffic": load_traffic(cfg_name), "pipe": pipe,
         "kernel": "k_update_tc (tcgen05 3xTF32 inner stage + level 0 + fp64 normal equations + Cholesky)" if tc
         else "k_update (fused TTV + fp64 normal equations + Cholesky)",
         "peak_source": {"fp32": f"derived: {nsm} SMs x 128 FMA/clk x 2 x {clk_mhz:.0f} MHz",
                         "fp64": f"derived: {nsm} SMs x 64 FMA/clk x 2 x {clk_mhz:.0f} MHz (pipe_probe: 63.2/clk measured)",
                         "tensor_f16": "MEASURED_PEAKS bf16_tflops (fp16 operands run at the bf16 rate)",
                         "hbm": "MEASURED_PEAKS hbm_gbs"}[pipe],
         "work_per_entry": {"fp32_fma": w32, "fp64_fma": w64, "tc_mac": wtc, "hbm_bytes": 4 * (N - 1) + sv},
         "roof_ms_by_pipe": {k: v * 1e3 for k, v in t.items()}, "roof_ms": t[pipe] * 1e3}
    if per_mode:
        r["per_mode"] = per_mode
        r["roof_ms"] = sum(m["roof_ms"] for m in per_mode)
        r["kernel"] = "k_update / k_update_smp2 / table k_update (per mode, SMP)"
    if xu:
        xu_peak = nsm * 16 * clk_mhz * 1e6
        r["xu_conversions_per_entry"] = xu
        r["xu_floor_ms"] = xu * entries / xu_peak * 1e3
    if tc:
        # one K sweep over [lo | hi | hi] padded to the f16 K-step of 16, N padded to 16
        kc, np_ = -(-(3 * J) // 16) * 16, -(-(J * J) // 16) * 16
        r["tc_executed_mac_per_entry"] = kc * np_
        r["tc_executed_floor_ms"] = 2 * kc * np_ * entries / (ptc * 1e12) * 1e3
    return r


def clocks_sampler(device: int):
    q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    try:
        return subprocess.Popen(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits", "-lms", "100",
                                 "-i", str(device)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
    except Exception:
        return None


def clocks_summary(proc):
    if proc is None:
        return None
    proc.terminate()
    try:
        out, _ = proc.communicate(timeout=5)
    except Exception:
        proc.kill()
        return None
    sm, mx, reasons = [], 0.0, set()
    names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
    for line in out.strip().splitlines():
        f = [x.strip() for x in line.split(",")]
        if len(f) < 8:
            continue
        try:
            sm.append(float(f[0]))
            mx = max(mx, float(f[1]))
        except ValueError:
            continue
        for nm, v in zip(names, f[4:8]):
            if v.lower() == "active":
                reasons.add(nm)
    if not sm:
        return None
    return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def load_traffic(cfg_name: str):
    """Per-launch DRAM bytes of the update kernel from the committed ncu capture, if any."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        d = json.load(open(p))
        return d.get(cfg_name)
    except Exception:
        return None


# ----------------------------------------------------------------------------- oracle arm
class OracleSample:
    """The FP64 CPU oracle (as it stands) on a bounded sample of the workload: for each
    mode n, the rows [0, R) of mode n with all their entries (a sub-tensor with I_n = R,
    the other dims unchanged, so rows keep the workload's length mix).  One sampled
    step = one oracle update_mode per mode plus the literal Eq. 5 error over the mode-0
    sample's entries -- the oracle's own full ALS iteration restricted to those rows.
    The sub-tensors and their slice indices are built once (like the GPU's index, outside
    the timed step)."""

    def __init__(self, cfg, coords, vals, R):
        from oracle import oracle as orc
        import multiprocessing
        self.orc, self.cfg, self.R = orc, cfg, R
        self.cores = multiprocessing.cpu_count()
        N, J = len(cfg.dims), cfg.J
        model = orc.init_model(cfg.dims, [J] * N, seed=cfg.seed, prec=1 if cfg.dtype == "f64" else 0)
        self.parts = []
        for n in range(N + 1):           # n = N: the error pass over the mode-0 sample
            m_ = 0 if n == N else n
            sel = coords[:, m_] < R
            dims = list(cfg.dims)
            dims[m_] = R
            t = orc.Tensor(np.ascontiguousarray(coords[sel]), vals[sel].astype(np.float64), dims)
            t.mode_index(m_)
            self.parts.append((n, t, orc.Model(model.G, [model.A(k)[:dims[k]] for k in range(N)])))
        self.entries = sum(t.nnz for n, t, _ in self.parts if n < N)   # entry-updates of the sampled iteration
        self.err_entries = self.parts[-1][1].nnz

    def step(self):
        """One sampled iteration; returns (seconds, entries/s by summed per-entry times)."""
        N = len(self.cfg.dims)
        took, per_entry = 0.0, 0.0
        for n, t, m in self.parts:
            t0 = time.perf_counter()
            if n < N:
                self.orc.update_mode(t, m, n, self.cfg.lam, threads=self.cores)
            else:
                self.orc.sse(t, m, threads=self.cores)
            dt = time.perf_counter() - t0
            took += dt
            per_entry += dt / max(t.nnz, 1)
        return took, 1.0 / per_entry

    def describe(self):
        N, nnz = len(self.cfg.dims), self.cfg.nnz
        return (f"oracle (FP64 C, OpenMP dynamic rows) on rows [0,{self.R}) of each mode with all their entries "
                f"({self.entries} entry-updates = {self.entries / (N * nnz):.4%} of the {N} x {nnz} of a full "
                f"iteration) + literal Eq.5 on the mode-0 sample ({self.err_entries} entries); entries/s from the "
                f"per-entry times summed over the {N} mode updates and the error pass")


def oracle_calibrated(cfg, coords, vals, target_s: float):
    """An OracleSample whose step takes about target_s seconds on this host."""
    R = max(8, min(cfg.dims) // 10000)
    s = OracleSample(cfg, coords, vals, R)
    took, _ = s.step()
    R2 = min(int(R * max(1.0, min(target_s / max(took, 1e-3), 1e4))), min(cfg.dims))
    if R2 > R:
        s = OracleSample(cfg, coords, vals, R2)
    return s


def oracle_sample_rate(cfg, coords, vals, target_s: float = 12.0):
    """cpu_baseline of our arm: one sampled oracle iteration of about target_s seconds.
    Returns (entries/s per full iteration, cores, description)."""
    s = oracle_calibrated(cfg, coords, vals, target_s)
    _, rate = s.step()
    return rate, s.cores, s.describe()


def run_reference(args, cfg):
    """--impl reference: the oracle arm.  Every step is one sampled oracle iteration
    (OracleSample) sized so the whole W + K run takes about args.ref_total seconds;
    ms_per_step is the measured time of those sampled steps (what ran), value is
    entries/s from the per-entry times, and `sample` states the fraction of a full
    iteration each step covers."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    coords, vals = synth.generate(cfg)
    per_step = max(0.5, min(args.ref_seconds, args.ref_total / max(args.warmup + args.steps, 1)))
    s = oracle_calibrated(cfg, coords, vals, per_step)
    times, rates = [], []
    t_run = time.perf_counter()
    for i in range(args.warmup + args.steps):
        took, r = s.step()
        if i >= args.warmup:
            times.append(took)
            rates.append(r)
    wall = time.perf_counter() - t_run
    v = float(statistics.median(rates))
    N = len(cfg.dims)
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * float(statistics.median(times)), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(cfg, args),
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": s.cores, "kind": "oracle", "sample": s.describe()},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "sample": {"rows_per_mode": s.R, "entry_updates_per_step": s.entries,
                   "fraction_of_full_iteration": s.entries / (N * cfg.nnz), "steps_timed": len(times),
                   "timed_wall_s": wall, "full_iteration_ms_extrapolated": 1e3 * cfg.nnz / v,
                   "note": "ms_per_step is the measured time of one SAMPLED iteration (rows [0,R) of every "
                           "mode); a full-size oracle iteration would take full_iteration_ms_extrapolated"},
    }
    print(json.dumps(line), flush=True)


def workload_config(cfg, args):
    return {
        "workload": f"{cfg.name}: order-{len(cfg.dims)} {'x'.join(str(d) for d in cfg.dims)}, |Omega|={cfg.nnz}, "
                    f"J={cfg.J}, lambda={cfg.lam}, values={cfg.values}, coords={cfg.coords}",
        "dims": list(cfg.dims), "nnz": cfg.nnz, "J": cfg.J, "lambda": cfg.lam, "seed": cfg.seed,
        "parallelism": f"rows of each mode sharded over {args.gpus} GPU(s); replicas refreshed by "
                       f"{'NVLink row pushes from the update kernels' if getattr(args, 'exchange', 'push') == 'push' else 'NCCL all-gather-v'} per mode",
        "l2": "inputs larger than L2 (no flush)",
    }


# ----------------------------------------------------------------------------- our arm
def open_peers(pt, dist, world, args):
    """Multi-GPU replica refresh by push: every rank opens the other
    ranks' factor replicas from their CUDA IPC handles; the update kernels then store
    each solved row into every replica over NVLink.  --exchange nccl keeps the NCCL
    all-gather-v instead."""
    pt.ptucker_set_option("exchange", 1 if args.exchange == "push" else 0)
    if world == 1 or args.exchange != "push":
        return
    hs = [None] * world
    dist.all_gather_object(hs, pt.ptucker_peer_handles())
    ok = True
    try:
        pt.ptucker_open_peers(b"".join(hs), world)
    except pt.PTuckerError as e:   # no peer access: the NCCL all-gather-v keeps the replicas fresh
        print(f"[bench] rank {dist.get_rank()}: peer replicas not opened ({e}); NCCL all-gather-v instead",
              file=sys.stderr, flush=True)
        ok = False
    flags = [None] * world
    dist.all_gather_object(flags, ok)
    if not all(flags):             # every rank must use the same exchange
        pt.ptucker_set_option("exchange", 0)


def run_ours(args, cfg):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_1710_02261_b200 import build, ptucker as pt
    if rank == 0 or world == 1:
        build.build()
    if world > 1:
        dist.barrier()
    pt.load()
    if world > 1:
        obj = [pt.ptucker_get_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        pt.ptucker_comm_init(rank, world, obj[0])
    # one dedicated stream for the library's kernels AND the timing events (torch's default
    # stream handle 0 would make the library create its own stream beside the events)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    pt.ptucker_set_stream(stream.cuda_stream)
    pt.ptucker_set_option("seg_len", args.seg_len)

    coords, vals = synth.generate(cfg)
    N, J = len(cfg.dims), cfg.J
    t0 = time.perf_counter()
    pt.ptucker_init(coords, vals, cfg.dims, [J] * N, cfg.lam, cfg.seed)
    pt.ptucker_set_option("policy", POLICY[args.policy])
    pt.ptucker_set_option("tc", args.tc)
    pt.ptucker_set_option("l0_group", args.l0_group)
    if args.l2_persist_mb is not None:
        pt.ptucker_set_option("l2_persist_mb", args.l2_persist_mb)
    pt.ptucker_set_option("pack_gathers", args.pack_gathers)
    for kv in args.opt:  # experiments: any library option (include/ptucker.h), e.g. fin_inline=0
        k, v = kv.split("=")
        pt.ptucker_set_option(k, int(v))
    open_peers(pt, dist, world, args)
    pt.ptucker_synchronize()
    init_s = time.perf_counter() - t0
    info = pt.ptucker_info()

    def barrier_sync():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        pt.ptucker_sweep()
        pt.ptucker_error()
        if args.approx > 0:
            pt.ptucker_truncate_core(args.approx)
    barrier_sync()
    # the timed loop runs as a user's would: sweeps replayed from the library's CUDA graph,
    # no per-kernel events; a second pass of the same length with kernel timing on gives the
    # per-kernel split for the roofline (its launches are serialised by the events)
    launches0 = pt.ptucker_info()["kernel_launches"]
    clk = clocks_sampler(local)
    time.sleep(0.3)
    errs = []
    barrier_sync()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        pt.ptucker_sweep()
        errs.append(pt.ptucker_error())
        if args.approx > 0:
            pt.ptucker_truncate_core(args.approx)  # P-Tucker-Approx: Alg. 2 lines 5-6
    ev1.record(stream)
    barrier_sync()
    clocks = clocks_summary(clk)
    ms = ev0.elapsed_time(ev1)
    launches = pt.ptucker_info()["kernel_launches"] - launches0
    # self-check state: the factors right after the timed loop
    import hashlib
    hsh = hashlib.sha256()
    for n in range(N):
        hsh.update(np.ascontiguousarray(pt.ptucker_get_factor(n)).tobytes())
    hsh.update(np.ascontiguousarray(pt.ptucker_get_core()).tobytes())
    # kernel-timing pass
    pt.ptucker_set_option("time_kernels", 1)
    pt.ptucker_reset_kernel_stats()
    barrier_sync()
    evp0 = torch.cuda.Event(enable_timing=True)
    evp1 = torch.cuda.Event(enable_timing=True)
    evp0.record(stream)
    for _ in range(args.steps):
        pt.ptucker_sweep()
        pt.ptucker_error()
        if args.approx > 0:
            pt.ptucker_truncate_core(args.approx)
    evp1.record(stream)
    barrier_sync()
    ms_profiled = evp0.elapsed_time(evp1)
    upd_ms, upd_n = pt.ptucker_kernel_stats("update")
    upd_ms_rank = upd_ms
    fin_ms, _ = pt.ptucker_kernel_stats("finalize")
    apx_ms, apx_n = pt.ptucker_kernel_stats("approx_scores") if args.approx > 0 else (0.0, 0)
    per_mode = {f"update_m{n}": round(pt.ptucker_kernel_stats(f"update_m{n}")[0] / args.steps, 4) for n in range(N)}
    per_mode.update({f"finalize_m{n}": round(pt.ptucker_kernel_stats(f"finalize_m{n}")[0] / args.steps, 4)
                     for n in range(N)})
    # multi-GPU self-check (F9: factors are bit-identical for any number of GPUs): a hash
    # of every A^(n) and of G after the timed run, the last error, the communicator size
    # and each rank's update / all-gather device time -- equal hashes and errors across
    # N = 1, 2, 4, 8 lines prove the exchange moved every row
    ag_ms, _ = pt.ptucker_kernel_stats("allgather")
    per_rank = [[upd_ms_rank / args.steps, ag_ms / args.steps]]
    if world > 1:
        t = torch.tensor(per_rank[0], dtype=torch.float64, device="cuda")
        allt = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(allt, t)
        per_rank = [x.tolist() for x in allt]
    selfcheck = {"factors_sha256": hsh.hexdigest()[:32], "last_error": errs[-1],
                 "comm_ranks": pt.ptucker_info()["comm_ranks"], "world": world,
                 "exchange": pt.ptucker_info()["exchange"],
                 "update_ms_per_step_by_rank": [round(x[0], 4) for x in per_rank],
                 "allgather_ms_per_step_by_rank": [round(x[1], 4) for x in per_rank]}

    pt.ptucker_set_option("time_kernels", 0)
    if world > 1:
        t = torch.tensor([ms, upd_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, upd_ms = float(t[0]), float(t[1])
    ms_per_step = ms / args.steps
    value = cfg.nnz * args.steps / (ms / 1e3)

    # roofline of the dominant kernel (the fused row update), per launch
    policy = info["policy"]
    nsm = torch.cuda.get_device_properties(local).multi_processor_count
    clk_max = (clocks or {}).get("sm_max_mhz") or 1965.0
    entries_per_launch = cfg.nnz / world           # each rank's launch covers its row block of one mode
    avg_launch_s = (upd_ms / max(upd_n, 1)) / 1e3
    mode_s = [per_mode[f"update_m{n}"] / 1e3 for n in range(N)]
    roof = roofline(N, J, policy, info, args.l0_group, nsm, clk_max, entries_per_launch, avg_launch_s,
                    cfg.dtype, cfg.name, mode_s)
    if args.approx > 0:
        roof["approx"] = {"p": args.approx, "scores_ms_per_step": apx_ms / args.steps,
                          "core_nnz_after": pt.ptucker_core_nnz()}
    roof.update({"avg_launch_ms": avg_launch_s * 1e3, "launches": upd_n, "update_share_of_step": upd_ms / ms_profiled,
                 "timing_pass_ms_per_step": ms_profiled / args.steps,
                 "finalize_ms_per_step": fin_ms / args.steps, "ms_per_step_by_kernel": per_mode})

    # e2e: the whole job through the public API from pinned host buffers
    e2e = None
    if not args.no_e2e:
        pc = torch.from_numpy(coords).pin_memory().numpy()
        pv = torch.from_numpy(vals).pin_memory().numpy()
        pt.ptucker_finalize()  # the previous context's teardown is not part of this job
        if world > 1:
            obj = [pt.ptucker_get_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            pt.ptucker_comm_init(rank, world, obj[0])
        pt.ptucker_set_option("seg_len", args.seg_len)
        barrier_sync()
        t0 = time.perf_counter()
        pt.ptucker_set_stream(stream.cuda_stream)
        pt.ptucker_init(pc, pv, cfg.dims, [J] * N, cfg.lam, cfg.seed)
        pt.ptucker_set_option("policy", POLICY[args.policy])
        pt.ptucker_set_option("tc", args.tc)
        pt.ptucker_set_option("l0_group", args.l0_group)
        open_peers(pt, dist, world, args)
        pt.ptucker_synchronize()
        t_init = time.perf_counter() - t0
        for _ in range(args.steps):
            pt.ptucker_sweep()
            pt.ptucker_error()
        barrier_sync()
        e2e_s = time.perf_counter() - t0
        if world > 1:
            t = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_s = float(t[0])
        e2e = {"value": cfg.nnz * args.steps / e2e_s, "unit": UNIT,
               "h2d_bytes_per_step": int((coords.nbytes + vals.nbytes) / args.steps), "d2h_bytes_per_step": 8,
               "init_s": t_init, "iterations_s": e2e_s - t_init,
               "note": f"ptucker_init from pinned host COO (H2D + validation + device index build) + {args.steps} "
                       f"iterations with the error read back each iteration; H2D amortised over the steps"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        r, cores, desc = oracle_sample_rate(cfg, coords, vals, target_s=args.ref_seconds)
        cpu = {"value": r, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": desc}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "fp32 storage/contraction + fp64 normal equations" if cfg.dtype == "f32"
            else "f64", "data": "synthetic", "config": workload_config(cfg, args) | {"policy": policy},
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clocks,
            "init_s": init_s, "errors": errs[-1:], "selfcheck": selfcheck, "info": {k: info[k] for k in ("grid_update", "seg_len", "tensor_cores", "modes")},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c5")
    ap.add_argument("--scale", type=float, default=1.0, help="shrink the config (tests only)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--policy", default="auto", choices=list(POLICY))
    ap.add_argument("--seg-len", type=int, default=-1, help="segment length S (-1 = the library's automatic choice)")
    ap.add_argument("--tc", type=int, default=1, choices=[0, 1], help="tensor-core inner stage for order-3 fp32")
    ap.add_argument("--l2-persist-mb", type=int, default=None,
                    help="L2 set-aside for evict_last accesses in MB (-1 = device maximum, the library's "
                         "default; 0 = leave the driver's setting)")
    ap.add_argument("--pack-gathers", type=int, default=0, choices=[0, 1],
                    help="J = 10 tensor-core gathers from packed 40-byte tables (less DRAM traffic, slower)")
    ap.add_argument("--l0-group", type=int, default=1, choices=[0, 1, 2, 5], help="tensor-core level-0 grouping (1 = fp64 per term, g = fp32 partial sums of g terms, 0 = compensated fp32 pairs)")
    ap.add_argument("--exchange", default="push", choices=["push", "nccl"],
                    help="multi-GPU replica refresh: rows pushed by the kernels over NVLink, or NCCL all-gather-v")
    ap.add_argument("--dtype", default=None, choices=["f32", "f64"],
                    help="storage precision override (default: the config's; f64 = the FP64 mode)")
    ap.add_argument("--approx", type=float, default=0.0,
                    help="P-Tucker-Approx: truncate the core by rate p after every iteration (0 = P-Tucker)")
    ap.add_argument("--ref-seconds", type=float, default=12.0, help="oracle seconds per sampled step (upper bound)")
    ap.add_argument("--ref-total", type=float, default=150.0, help="reference arm: seconds for all W + K sampled steps")
    ap.add_argument("--opt", action="append", default=[], help="library option key=value (repeatable; experiments)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    cfg = synth.config(args.config) if args.scale == 1.0 else synth.small(args.config, args.scale)
    if args.dtype:   # FP64 mode of a config (values, factors and core stored in fp64: 1e-10 parity class)
        import dataclasses
        cfg = dataclasses.replace(cfg, dtype=args.dtype)
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
