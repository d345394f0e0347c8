#!/usr/bin/env python
"""Benchmark: tokens/s for forward+backward of ONE LSS attention layer
(l_x = 50112, E_m = 1024, 16 heads, causal, bf16 operands / fp32 accumulation)
on N B200s of one node, N = 1, 2, 4, 8 (BASELINE.json `metric`).

    python bench.py [--gpus N --steps K --warmup W]               # our B200 path
    python bench.py --impl reference [...]                          # reference CPU arm
    torchrun --nproc-per-node N bench.py --gpus N ...               # N > 1 (NCCL)

A step = the attention sublayer of one layer: LN1, [Q|K|V] projection,
packed-K/V all-gather, segment attention, out-projection + residual, and the
whole backward incl. the dK/dV reduce-scatter and the folded gradient
all-reduce, plus the per-step weight staging.  The sequence is split across the
N ranks (ShardSpec), so total work is fixed: scaling = "strong".  Synthetic
inputs (x, upstream gradient ~ N(0,1)) and random-init weights of the named
shape (U(+-1/sqrt(E)), zero biases, unit LN gain -- model.init_params's
convention).  The per-step working set (>= 0.6 GB of K/V and dK/dV buffers)
is larger than the 126 MB L2, so no explicit flush is needed.
"""

from __future__ import annotations

import argparse
import dataclasses
import json
import math
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "tokens/sec fwd+bwd per LSS attention layer at l_x=50112, 1/2/4/8 B200; % bf16 peak"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--seq", type=int, default=50112)
    ap.add_argument("--embed", type=int, default=1024)
    ap.add_argument("--heads", type=int, default=16)
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--noncausal", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-rows", type=int, default=128, help="query rows in the CPU sample")
    ap.add_argument("--unbalanced", action="store_true", help="plain contiguous causal schedule")
    ap.add_argument("--model", choices=["layer", "gpt"], default="layer",
                    help="layer: the BASELINE metric (one LSS attention layer); gpt: the L-layer decoder "
                         "training step of BASELINE configs 4/5 (embedding, L complete layers, head, loss, "
                         "one all-reduce, SGD update)")
    ap.add_argument("--layers", type=int, default=12)
    ap.add_argument("--replicas", type=int, default=1, help="gpt: data-parallel replicas D (world = D x N)")
    return ap.parse_args()


def workload(args):
    return (f"LSS attention sublayer fwd+bwd, l_x={args.seq}, E_m={args.embed}, {args.heads} heads, "
            f"{'non-causal' if args.noncausal else 'causal'}, batch {args.batch}")


def layer_flops(batch, seq, embed, causal):
    """F = 24 l E^2 + 12 E P per sequence, P = l(l+1)/2 causal or l^2."""
    pairs = seq * (seq + 1) // 2 if causal else seq * seq
    return batch * (24 * seq * embed * embed + 12 * embed * pairs)


def rank_pairs(offset, rows, seq, causal):
    """Unmasked (q, k) pairs of query rows [offset, offset+rows) against seq keys."""
    if not causal:
        return rows * seq
    full = max(0, min(rows, seq - offset))  # rows whose key range ends inside the sequence
    return full * offset + full * (full + 1) // 2 + (rows - full) * seq


def peaks():
    try:
        d = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
        return float(d["bf16_tflops"]), float(d["bf16_tflops_sustained"]), "measured"
    except Exception:
        return 1590.0, 1400.0, "fallback"


def traffic_from_profile(name):
    """dram bytes per launch of `name` from the committed ncu --set full summary, if any."""
    p = ROOT / "profiles" / "ncu_summary.json"
    try:
        d = json.loads(p.read_text())
        return d["kernels"][name]["dram_bytes_per_launch"]
    except Exception:
        return None


# ------------------------------------------------------------------ clocks


class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index):
        self.proc = None
        self.t0 = self.t1 = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "100",
                 "-i", str(device_index)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        self.lines = []

    def start(self):
        self.t0 = time.time()

    def stop(self):
        self.t1 = time.time()
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=5)
        rows = [ln.split(", ") for ln in out.strip().splitlines() if ln.strip()]
        sm = [float(r[1]) for r in rows if len(r) >= 9 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if len(r) >= 9 and r[2].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            if len(r) < 9:
                continue
            for nm, val in zip(names, r[5:9]):
                if val.strip().lower() == "active":
                    reasons.add(nm)
        # the sampler runs a little before/after the timed region: keep the loaded samples
        loaded = [s for s in sm if s > 0.5 * max(sm)] if sm else []
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------------ reference / CPU arm


def host_info(kind="port"):
    """CPU model, numpy and BLAS of the host the CPU legs ran on."""
    import platform

    import numpy as np

    model = platform.processor() or "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    blas = "unknown"
    try:
        b = np.show_config(mode="dicts")["Build Dependencies"]["blas"]
        blas = f"{b.get('name')} {b.get('version')}"
    except Exception:  # noqa: BLE001 - informational only
        pass
    prec = ("the reference's own 'single' path (scores and softmax promoted to fp64 under NumPy 2, SURVEY §0.7)"
            if kind == "reference" else "fp32 numpy port of the reference's functions (oracle/lss_oracle.py)")
    return {"cpu_model": model, "host_cpus": os.cpu_count(), "numpy": np.__version__, "blas": blas,
            "precision": prec}



def cpu_sample(args, rows, threads):
    """Time the oracle port of the reference's attention sublayer on a bounded
    sample: `rows` query rows centred on l/2 (the mean causal row) against the
    full-length K/V.  Returns (seconds, description)."""
    import numpy as np

    from oracle import lss_oracle as O

    rng = np.random.default_rng(0)
    x = rng.standard_normal((args.batch, args.seq, args.embed), dtype=np.float32)
    gy = rng.standard_normal((args.batch, args.seq, args.embed), dtype=np.float32)
    p = O.init_attn_params(args.embed, seed=0, dtype=np.float32)
    offset = max(0, args.seq // 2 - rows // 2)
    run = O.sample_rows(x, gy, p, args.heads, offset, rows, causal=not args.noncausal)
    return run, (f"{rows} query rows at offset {offset} of l_x={args.seq} (fp32 numpy oracle port of the "
                 f"reference's scores_fwd/scores_bwd + projections + LN; K/V of the whole sequence "
                 f"precomputed), {threads} host threads")


REF_INSTALL = ROOT / "baseline" / "_ref"


def reference_sample(args, rows, threads):
    """Time the REFERENCE's own functions (seqpar, installed under baseline/_ref by
    ``pip install --target``) on a bounded sample: ``rows`` query rows centred on
    l/2 through the attention half of model.layer_fwd / layer_bwd -- norm3, linear3
    (Q and own K/V), scores_fwd / scores_bwd (its per-(sample, head) loop with the
    full probability matrix, model.py:280-359), the out-projection, linear3_bwd x4
    and norm3_bwd -- against the K/V of the whole sequence (projected outside the
    timed region, as if received from the all-gather).  precision "single", the
    reference's fp32 mode.  Returns (run, description) or None when absent."""
    if not (REF_INSTALL / "seqpar").exists():
        return None
    sys.path.insert(0, str(REF_INSTALL))
    import numpy as np
    from seqpar import model as RM
    from seqpar.nnops import DropoutPolicy

    cfg = RM.ModelConfig(embed_dim=args.embed, n_layers=1, n_heads=args.heads, ff_dim=4, vocab=16,
                         seq_len=args.seq, batch=args.batch, causal=not args.noncausal, precision="single")
    lp = RM.init_params(RM.ModelConfig(**{**cfg.to_dict(), "seq_len": 8}), 0).layers[0]
    rng = np.random.default_rng(0)
    x = rng.standard_normal((args.batch, args.seq, args.embed), dtype=np.float32)
    gy = rng.standard_normal((args.batch, rows, args.embed), dtype=np.float32)
    offset = max(0, args.seq // 2 - rows // 2)
    xh_all, _ = RM.norm3(x, lp.ln1_gain, lp.ln1_bias)
    k_full, v_full = RM.linear3(xh_all, lp.attn_k), RM.linear3(xh_all, lp.attn_v)
    off = DropoutPolicy.off()
    xs = np.ascontiguousarray(x[:, offset:offset + rows])

    def run():
        xh, ln = RM.norm3(xs, lp.ln1_gain, lp.ln1_bias)
        k_own, v_own = RM.linear3(xh, lp.attn_k), RM.linear3(xh, lp.attn_v)
        q = RM.linear3(xh, lp.attn_q)
        ctx, sc = RM.scores_fwd(q, k_full, v_full, offset, cfg, off, 0)
        y = xs + RM.linear3(ctx, lp.attn_out)
        g_ctx, _, _ = RM.linear3_bwd(ctx, lp.attn_out, gy)
        dq, dk, dv = RM.scores_bwd(sc, q, k_full, v_full, g_ctx, cfg, off)
        gxq, _, _ = RM.linear3_bwd(xh, lp.attn_q, dq)
        gxk, _, _ = RM.linear3_bwd(xh, lp.attn_k, dk[:, offset:offset + rows])
        gxv, _, _ = RM.linear3_bwd(xh, lp.attn_v, dv[:, offset:offset + rows])
        gx, _, _ = RM.norm3_bwd(ln, lp.ln1_gain, gxq + gxk + gxv)
        return y, gy + gx, k_own, v_own

    return run, (f"{rows} query rows at offset {offset} of l_x={args.seq} through the REFERENCE's own "
                 f"seqpar functions (baseline/_ref; norm3, linear3, scores_fwd/scores_bwd, linear3_bwd, "
                 f"norm3_bwd; precision 'single'), K/V of the whole sequence precomputed; {threads} host "
                 f"threads available to its BLAS")


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    threads = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    rows = max(8, min(args.cpu_rows, 64))
    ref = reference_sample(args, rows, threads)
    kind = "reference" if ref is not None else "port"
    run, desc = ref if ref is not None else cpu_sample(args, rows, threads)
    for _ in range(args.warmup):
        run()
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        run()
        times.append(time.perf_counter() - t0)
    t = statistics.median(times)
    value = args.batch * rows / t
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": workload(args), "global_batch": args.batch, "seq_len": args.seq,
                   "parallelism": "cpu"},
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": threads, "kind": kind,
                         "sample": desc, **host_info(kind)},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    emit(line)
    return 0


# ------------------------------------------------------------------ our arm


def main_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2311_02382_b200 import _native
    from paper_2311_02382_b200.comm import Ledger, SoloComm, TorchDistComm
    from paper_2311_02382_b200.model import LayerParams, LinearParams, ModelConfig
    from paper_2311_02382_b200.sharded import EngineOptions, LSSAttention, ShardSpec

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        # stream-wait mode for A/B runs (default "kernel"; "guarded" / "frontend")
        comm = TorchDistComm(None, None, Ledger(), bounded_waits=os.environ.get("LSS_WAITS", "kernel"))
    else:
        comm = SoloComm(Ledger())
    causal = not args.noncausal
    B, l, E, H = args.batch, args.seq, args.embed, args.heads
    cfg = ModelConfig(embed_dim=E, n_layers=1, n_heads=H, ff_dim=4 * E, vocab=256, seq_len=l, batch=B,
                      causal=causal, precision="bf16")
    spec = ShardSpec(rank, world, l)
    m = spec.block
    g = torch.Generator(device=dev).manual_seed(1234)
    bound = 1.0 / math.sqrt(E)
    u = lambda: (torch.rand(E, E, generator=g, device=dev) * 2 - 1) * bound  # noqa: E731
    z = lambda: torch.zeros(E, device=dev)  # noqa: E731
    lp = LayerParams(torch.ones(E, device=dev), z(), LinearParams(u(), z()), LinearParams(u(), z()),
                     LinearParams(u(), z()), LinearParams(u(), z()))
    gx = torch.Generator(device=dev).manual_seed(100 + rank)
    x = torch.randn(B, m, E, generator=gx, device=dev)
    gy = torch.randn(B, m, E, generator=gx, device=dev)
    # execution options: the production defaults, overridable for A/B runs by LSS_* variables read HERE
    # (explicitly; the package itself never reads the environment)
    opts = EngineOptions.from_env()
    if args.unbalanced:
        opts = dataclasses.replace(opts, balanced=False)
    eng = LSSAttention(cfg, spec, grad_scale=1.0 / world, device=dev, options=opts)

    # per-kernel CUDA-event timing of the two attention kernels inside the timed region
    stream = torch.cuda.current_stream()
    marks = {"fwd": [], "bwd": []}
    from paper_2311_02382_b200 import kernels as Kmod

    wrapped = {"attn_fwd": "fwd", "attn_fwd_partial": "fwd", "attn_bwd": "bwd", "attn_bwd_sources": "bwd",
               "gemm": "qkv"}
    marks["qkv"] = []
    originals = {name: getattr(Kmod, name) for name in wrapped}

    def timed(kind, fn):
        def wrapper(*a, **kw):
            if kind == "qkv" and not (kw.get("N") == 3 * E and kw.get("K") == E and kw.get("M") == B * m):
                return fn(*a, **kw)  # only the [Q|K|V] projection GEMM is timed
            # on the stream the launch goes to (side streams at N > 1: fused gather,
            # delegated rows); concurrent launches are summed, so the figure is conservative
            st = torch.cuda.current_stream()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(st)
            out = fn(*a, **kw)
            e1.record(st)
            marks[kind].append((e0, e1, cur_step[0]))
            return out
        return wrapper

    cur_step = [0]

    def one_step():
        cur_step[0] += 1
        eng.load_params(lp)  # weights change every training step: restage (1 kernel)
        eng.step(x, gy, comm)

    for _ in range(args.warmup):
        one_step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    for name, kind in wrapped.items():
        setattr(Kmod, name, timed(kind, originals[name]))
    sampler = ClockSampler(local)
    time.sleep(0.3)  # let the sampler come up
    comm.ledger.clear()
    launches0 = _native.launch_count
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    sampler.start()
    t_start.record(stream)
    for _ in range(args.steps):
        one_step()
    t_end.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = sampler.stop()
    for name in wrapped:
        setattr(Kmod, name, originals[name])
    launches = (_native.launch_count - launches0) // args.steps
    if opts.phases in (1, 2):  # diagnostic: one extra step with a per-phase timeline
        from paper_2311_02382_b200 import engine as _sh
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        one_step()
        if opts.phases == 2:  # steady state: back-to-back steps, stamps of the last
            for _ in range(4):
                one_step()
            _sh.last_phases = _sh.last_clock.report()
        ph = {k: round(v, 3) for k, v in _sh.last_phases.items()}
        if _sh.last_stamps and world > 1:  # cross-rank timeline (GPU global timer, us after the earliest start)
            allst = [None] * world
            dist.all_gather_object(allst, _sh.last_stamps)
            if rank == 0:  # per-GPU timers are not synchronised: align on the backward barrier's release
                names = [n for n, _ in allst[0]]
                ai = names.index("rs_barrier") if "rs_barrier" in names else 0
                for i, name in enumerate(names):
                    print(f"[timeline] {name:16s} " + " ".join(f"{(st[i][1] - st[ai][1]) / 1e3:9.1f}"
                                                          for st in allst), file=sys.stderr, flush=True)
        torch.cuda.synchronize()
        eng.options = dataclasses.replace(eng.options, phases=0)  # the phase clock synchronises
        h0 = time.perf_counter()
        for _ in range(3):
            one_step()
        h1 = time.perf_counter()
        torch.cuda.synchronize()
        h2 = time.perf_counter()
        ph["host_enqueue_ms"] = round((h1 - h0) / 3 * 1e3, 3)
        ph["host_total_ms"] = round((h2 - h0) / 3 * 1e3, 3)
        print(f"[phases rank {rank}] " + json.dumps(ph), file=sys.stderr, flush=True)
    coll = {k: comm.ledger.count(k) // args.steps for k in ("all-gather", "reduce-scatter", "all-reduce")}
    ms = t_start.elapsed_time(t_end) / args.steps
    # per-step device time of this rank's attention kernels (all launches of the step)
    fwd_ms = sum(a.elapsed_time(b) for a, b, _ in marks["fwd"]) / args.steps
    bwd_ms = sum(a.elapsed_time(b) for a, b, _ in marks["bwd"]) / args.steps
    qkv_ms = sum(a.elapsed_time(b) for a, b, _ in marks["qkv"]) / max(1, len(marks["qkv"]))

    def span_ms(kind):
        """Per step, first launch start to last launch end of the kind's launches (at N > 1
        several launches run concurrently on side streams); mean over the timed steps."""
        steps = {}
        for a, b, k in marks[kind]:
            lo, hi = t_start.elapsed_time(a), t_start.elapsed_time(b)
            s0, s1 = steps.get(k, (lo, hi))
            steps[k] = (min(s0, lo), max(s1, hi))
        return sum(h - l_ for l_, h in steps.values()) / max(1, len(steps))

    my_pairs = eng.computed_pairs() * B
    stats = torch.tensor([ms, fwd_ms, bwd_ms, float(my_pairs), qkv_ms, span_ms("fwd"), span_ms("bwd")],
                         dtype=torch.float64, device=dev)
    if world > 1:
        allst = [torch.zeros_like(stats) for _ in range(world)]
        dist.all_gather(allst, stats)
        allst = torch.stack(allst).cpu().tolist()
    else:
        allst = [stats.cpu().tolist()]
    ms_max = max(r[0] for r in allst)
    crit = max(allst, key=lambda r: r[2])  # rank with the slowest attention backward
    tokens = B * l
    value = tokens / (ms_max / 1e3)
    burst, sustained, src = peaks()
    # the burst peak applies while the SMs run at their maximum clock; a power-capped run
    # whose loaded clock sits well below it is held to the sustained figure
    at_max = bool(clocks.get("sm_mhz") and clocks.get("sm_max_mhz") and clocks["sm_mhz"] >= 0.95 * clocks["sm_max_mhz"])
    peak, peak_name = (burst, "bf16_tflops (burst)") if at_max else (sustained, "bf16_tflops_sustained")
    total_flops = layer_flops(B, l, E, causal)
    pct = {"burst": total_flops / (ms_max / 1e3) / (world * burst * 1e12),
           "sustained": total_flops / (ms_max / 1e3) / (world * sustained * 1e12)}
    bwd_flops = 8 * E * crit[3]
    fwd_flops = 4 * E * crit[3]
    qkv_flops = 2 * (B * m) * (3 * E) * E
    ach_bwd = bwd_flops / (crit[2] / 1e3) / 1e12
    ach_fwd = fwd_flops / (crit[1] / 1e3) / 1e12
    ach_qkv = qkv_flops / (crit[4] / 1e3) / 1e12 if crit[4] > 0 else None

    def entry(kernel, ach, ms_k, work, traffic_key, flops=None, span=None):
        e = {"kernel": kernel, "bound": "tensor", "achieved": ach, "peak": peak, "unit": "TFLOP/s",
             "frac": ach / peak if ach else None, "frac_of_burst": ach / burst if ach else None,
             "frac_of_sustained": ach / sustained if ach else None, "ms_per_step": ms_k, "algorithmic": work,
             "traffic": traffic_from_profile(traffic_key), "traffic_source": "profiles/ncu_summary.json "
             "(dram__bytes_read.sum + dram__bytes_write.sum per launch, one ncu --set full capture)"}
        if flops and span and world > 1:
            # ms_per_step sums the launches of a step, which overlap on side streams at N > 1
            # (own rows, delegated rows, key splits): the span from the first start to the last
            # end is the time the phase actually occupies the GPU (fused-gather waits included)
            e.update(span_ms_per_step=span, frac_span=flops / (span / 1e3) / 1e12 / peak)
        return e

    roofline = entry("attn_bwd_tc_kernel (+ delta pre-pass)", ach_bwd, crit[2],
                     f"8*E per unmasked (q,k) pair; {crit[3]:.4g} pairs on the critical rank", "attn_bwd_tc_kernel",
                     bwd_flops, crit[6])
    roofline.update(peak_source=f"{src} {peak_name} (loaded SM clock {clocks.get('sm_mhz')} of "
                                f"{clocks.get('sm_max_mhz')} MHz)",
                    balanced_schedule=eng.plan.role != "none" or world == 1,
                    fwd=entry("attn_fwd_tc_kernel", ach_fwd, crit[1], "4*E per unmasked (q,k) pair", "attn_fwd_tc_kernel",
                              fwd_flops, crit[5]),
                    qkv_gemm=entry("gemm_bf16_tc_kernel<0,0> ([Q|K|V] projection)", ach_qkv, crit[4],
                                   f"2*M*N*K, M={B * m}, N={3 * E}, K={E} per launch", "gemm_qkv"))

    # ---------------- end-to-end through the public API with pinned host buffers
    e2e = None
    if not args.no_e2e:
        xh = x.cpu().pin_memory()
        gyh = gy.cpu().pin_memory()
        grads_h = torch.empty(eng.grads.numel(), dtype=torch.float32).pin_memory()
        for _ in range(2):
            eng.load_params(lp)
            eng.step_from_host(xh, gyh, comm, grads_h)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for i in range(args.steps):  # input prefetch: step i+1's H2D overlaps step i (one copy per step)
            eng.load_params(lp)
            eng.step_from_host(xh, gyh, comm, grads_h, next_inputs=(xh, gyh) if i + 1 < args.steps else None)
        stream.wait_event(eng.host_sync_event())  # every step's gradients are back on the host
        e1.record(stream)
        torch.cuda.synchronize()
        t_e2e = torch.tensor([e0.elapsed_time(e1) / args.steps], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t_e2e, op=dist.ReduceOp.MAX)
        e2e = {"value": tokens / (t_e2e.item() / 1e3), "unit": "tokens/s",
               "h2d_bytes_per_step": 2 * B * m * E * 4, "d2h_bytes_per_step": eng.grads.numel() * 4,
               "ms_per_step": t_e2e.item(),
               "api": "LSSAttention.step_from_host (pinned x, grad_y in, double-buffered with the next "
                      "step's copy overlapping this step; averaged grads out)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = len(os.sched_getaffinity(0))
        ref = reference_sample(args, args.cpu_rows, threads)
        kind = "reference" if ref is not None else "port"
        run, desc = ref if ref is not None else cpu_sample(args, args.cpu_rows, threads)
        run()  # warm
        reps, t0 = 0, time.perf_counter()
        while True:  # >= 10 s of CPU work (bounded sample, repeated)
            run()
            reps += 1
            dt = time.perf_counter() - t0
            if dt >= 10.0 or reps >= 50:
                break
        cpu = {"value": B * args.cpu_rows * reps / dt, "unit": "tokens/s", "cores": threads, "kind": kind,
               "sample": f"{reps} x " + desc, "seconds": dt, **host_info(kind)}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": workload(args), "global_batch": B, "seq_len": l, "embed": E,
                       "heads": H, "parallelism": f"sp{world}", "tokens_per_gpu": m,
                       "l2": "inputs larger than L2 (no flush)"},
            "pct_bf16_peak": pct,
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clocks,
            "per_rank_ms": [r[0] for r in allst],
            "collectives_per_step": coll,
        }
        emit(line)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main_gpt(args):
    """BASELINE configs 4/5: the L-layer decoder training step on a D x N grid."""
    import torch
    import torch.distributed as dist

    from paper_2311_02382_b200 import optim
    from paper_2311_02382_b200.comm import Ledger, SimComm, SoloComm, TorchDistComm
    from paper_2311_02382_b200.gpt import GPTRank, gpt_step
    from paper_2311_02382_b200.hybrid import GridLayout, make_groups
    from paper_2311_02382_b200.model import LayerParams, LinearParams, ModelConfig, Parameters
    from paper_2311_02382_b200.sharded import ShardSpec

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    lay = GridLayout(args.replicas, world // args.replicas)
    replica, seq_index = lay.coords(rank)
    data_comm = None
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        if args.replicas > 1:
            seq_g, data_g, world_g = make_groups(lay)
            comm = TorchDistComm(seq_g, world_g, Ledger())
            data_comm = TorchDistComm(data_g, data_g, Ledger())
        else:
            comm = TorchDistComm(None, None, Ledger())
    else:
        comm = SoloComm(Ledger())
    B, l, E, H, L, V = args.batch, args.seq, args.embed, args.heads, args.layers, 256
    F = 4 * E
    cfg = ModelConfig(embed_dim=E, n_layers=L, n_heads=H, ff_dim=F, vocab=V, seq_len=l, batch=B,
                      causal=not args.noncausal, precision="bf16")
    g = torch.Generator(device=dev).manual_seed(7)
    u = lambda a, b_: ((torch.rand(a, b_, generator=g, device=dev) * 2 - 1) / math.sqrt(a))  # noqa: E731
    z = lambda n: torch.zeros(n, device=dev)  # noqa: E731
    layers = [LayerParams(torch.ones(E, device=dev), z(E), LinearParams(u(E, E), z(E)), LinearParams(u(E, E), z(E)),
                          LinearParams(u(E, E), z(E)), LinearParams(u(E, E), z(E)), torch.ones(E, device=dev), z(E),
                          LinearParams(u(E, F), z(F)), LinearParams(u(F, E), z(E))) for _ in range(L)]
    spec = ShardSpec(seq_index, lay.seq_workers, l)
    P = Parameters(torch.randn(V, E, generator=g, device=dev) * 0.02,
                   torch.randn(spec.block, E, generator=g, device=dev) * 0.02, layers, torch.ones(E, device=dev),
                   z(E), LinearParams(u(E, V), z(V)))
    rk = GPTRank(cfg, spec, replicas=args.replicas, device=dev)
    rk.bind_params(P)
    del P, layers
    gt = torch.Generator(device=dev).manual_seed(100 + replica)
    tok = torch.randint(0, V, (B, l), generator=gt, device=dev)
    o, m = spec.offset, spec.block
    tseg, yseg = tok[:, o:o + m].contiguous(), torch.roll(tok, -1, 1)[:, o:o + m].contiguous()
    opt, opt_pos = optim.SGD(1e-4), optim.SGD(1e-4)

    def one_step():
        gpt_step([rk], comm, [tseg], [yseg], data_comm=data_comm)
        rk.optimizer_step(opt, opt_pos)

    for _ in range(args.warmup):
        one_step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    sampler = ClockSampler(local)
    time.sleep(0.3)
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sampler.start()
    e0.record(stream)
    for _ in range(args.steps):
        one_step()
    e1.record(stream)
    torch.cuda.synchronize()
    clocks = sampler.stop()
    t = torch.tensor([e0.elapsed_time(e1) / args.steps], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = t.item()
    loss = float(rk.loss())
    tokens = args.replicas * B * l
    pairs = l * (l + 1) // 2 if cfg.causal else l * l
    flops = args.replicas * B * (L * (24 * l * E * E + 12 * E * pairs + 12 * l * E * F) + 6 * l * E * V)
    burst, sustained, src = peaks()
    if rank == 0:
        line = {"metric": f"tokens/sec training step of the {L}-layer LSS decoder (embedding, layers, head, loss, "
                          "one all-reduce, SGD)", "value": tokens / (ms / 1e3), "unit": "tokens/s",
                "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
                "data": "synthetic", "config": {"workload": f"decoder L={L}, l_x={l}, E_m={E}, {H} heads, ff={F}, "
                                                            f"vocab {V}, batch {B}, grid {args.replicas}x{lay.seq_workers}",
                                                "parallelism": f"dp{args.replicas}xsp{lay.seq_workers}"},
                "pct_bf16_peak": {"burst": flops / (ms / 1e3) / (world * burst * 1e12),
                                  "sustained": flops / (ms / 1e3) / (world * sustained * 1e12)},
                "loss": loss, "clocks": clocks}
        emit(line)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


_JSON_OUT = None


def claim_stdout():
    """Route fd 1 to stderr for the rest of the run and keep the real stdout for the
    one JSON line: native libraries (NCCL's version banner on rank 0) print to fd 1."""
    global _JSON_OUT
    sys.stdout.flush()
    _JSON_OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)


def emit(line):
    print(json.dumps(line), file=_JSON_OUT or sys.stdout, flush=True)


def main():
    claim_stdout()
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    if args.model == "gpt":
        return main_gpt(args)
    return main_ours(args)


if __name__ == "__main__":
    sys.exit(main())
