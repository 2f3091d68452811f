#!/usr/bin/env python
"""Benchmark of the multipoint Kronecker-substitution hot path on B200.

Metric (BASELINE.json): polynomial products per second per KS variant, with
the multiply kernel's fraction of its measured peak: the dense tcgen05 u8 MMA
rate when it runs on the tensor cores (kmx_tc.cu), the IMAD.WIDE.U32 rate
when it runs on the integer pipe (kmx_mul.cu).
Default workload = BASELINE config 2 (configs[1]): Z[x], signed int32
coefficients, batch 1024 pairs, n = 1024.  A step = one pass of the hot path
(pack -> multiply -> finish [-> reconstruct] -> bias) over the whole batch.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c1|c2|c3|c4]
                  [--variant 1..4] [--impl ours|reference]

One JSON line on rank 0.  N > 1 runs under torchrun: every rank multiplies
its own batch (independent pairs, no collective on the data path: weak
scaling); the step time is the max over ranks.  ``--impl reference`` times the
reference algorithm's CPU implementation (the oracle port of kronmul, since
the reference is pure Python and /root/reference is absent on the GPU box)
on all host cores of rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "poly products/sec per KS variant; fraction of the tensor (or IMAD) peak and HBM roofline"
VNAME = {1: "ks1", 2: "ks2", 3: "ks3", 4: "ks4"}
VDESC = {1: "standard 2^N", 2: "reciprocal 2^N,2^-N", 3: "negated +-2^N", 4: "four-point +-2^N,+-2^-N"}
CONFIGS = {
    "c1": dict(kind="ks", batch=64, n=256, b=64, signed=False, seed=1,
               desc="c1: Z[x] u64 coefficients, batch 64, n=256"),
    "c2": dict(kind="ks", batch=1024, n=1024, b=32, signed=True, seed=2,
               desc="c2: Z[x] signed int32 coefficients, batch 1024, n=1024"),
    "c3": dict(kind="bks", batch=256, lx=64, ly=64, b=16, seed=3,
               desc="c3: R[x,y]->R[x], R=Z, u16 64x64 grids, batch 256"),
    "c4": dict(kind="ks", batch=32, n=4096, b=128, signed=False, seed=4,
               desc="c4: Z[x] u128 coefficients, batch 32, n=4096"),
}
L2_FLUSH_BYTES = 256 << 20


# ------------------------------------------------------------------ inputs
def make_inputs(cfg, rank=0):
    """Seeded numpy PCG64 inputs; words are little-endian u32."""
    import numpy as np
    rng = np.random.Generator(np.random.PCG64(cfg["seed"] * 1000 + rank))
    if cfg["kind"] == "bks":
        shp = (cfg["batch"], cfg["lx"], cfg["ly"])
        f = rng.integers(0, 1 << cfg["b"], size=shp, dtype=np.int64).astype(np.int32)
        g = rng.integers(0, 1 << cfg["b"], size=shp, dtype=np.int64).astype(np.int32)
        return f, g
    B, n, b = cfg["batch"], cfg["n"], cfg["b"]
    if cfg["signed"]:
        f = rng.integers(-(1 << (b - 1)), 1 << (b - 1), size=(B, n, 1), dtype=np.int64).astype(np.int32)
        g = rng.integers(-(1 << (b - 1)), 1 << (b - 1), size=(B, n, 1), dtype=np.int64).astype(np.int32)
        return f.view(np.uint32), g.view(np.uint32)
    words = (b + 31) // 32
    f = rng.integers(0, 1 << 32, size=(B, n, words), dtype=np.uint64).astype(np.uint32)
    g = rng.integers(0, 1 << 32, size=(B, n, words), dtype=np.uint64).astype(np.uint32)
    top = b - 32 * (words - 1)
    if top < 32:
        f[:, :, -1] &= (1 << top) - 1
        g[:, :, -1] &= (1 << top) - 1
    return f, g


def to_ints(arr, signed):
    import numpy as np
    a = np.ascontiguousarray(arr)
    if signed:
        return [[int(x) for x in row[:, 0].view(np.int32)] for row in a]
    out = []
    w = a.shape[2]
    for row in a:
        raw = row.astype(np.uint32).tobytes()
        out.append([int.from_bytes(raw[i:i + 4 * w], "little") for i in range(0, len(raw), 4 * w)])
    return out


def algorithmic_products(cfg, variant):
    """Schoolbook 32x32 limb products per pair: sum over the
    sub-products of m_f * m_g, m = ceil((N (L-1) + b + 2) / 32) limbs."""
    import ctypes
    from paper_0712_4046_b200 import _lib
    if cfg["kind"] == "bks":
        lx, ly = cfg["lx"], cfg["ly"]
        Lu = {1: (2 * lx - 1) * (ly - 1) + lx, 2: lx * ly, 3: lx * ly, 4: (lx + 1) // 2 * (ly - 1) + lx}[variant]
        P = {1: 1, 2: 2, 3: 2, 4: 4}[variant]
        return P * Lu * Lu
    p = (ctypes.c_int64 * 8)()
    flags = _lib.KMX_SIGNED if cfg["signed"] else 0
    _lib.check(_lib.lib().kmx_ks_params(variant, cfg["n"], cfg["n"], cfg["b"], flags, p))
    eff_variant = variant
    if variant == 4 and (not p[4] or p[5] == 1):
        eff_variant = 1
    P = {1: 1, 2: 2, 3: 2, 4: 4}[eff_variant]
    return P * int(p[6]) * int(p[7])


def pack_unpack_bytes(cfg, variant):
    """Algorithmic HBM bytes of one step outside the multiply: inputs + packed
    operands (pack), products + outputs (finish), digit streams (recon)."""
    import ctypes
    from paper_0712_4046_b200 import _lib
    if cfg["kind"] == "bks":
        return None
    p = (ctypes.c_int64 * 8)()
    flags = _lib.KMX_SIGNED if cfg["signed"] else 0
    _lib.check(_lib.lib().kmx_ks_params(variant, cfg["n"], cfg["n"], cfg["b"], flags, p))
    P = {1: 1, 2: 2, 3: 2, 4: 4}[variant]
    B, n = cfg["batch"], cfg["n"]
    iw = 1 if cfg["signed"] else (cfg["b"] + 31) // 32
    ow = _lib.lib().kmx_ks_out_words(n, n, cfg["b"], flags)
    mf, mg = int(p[6]), int(p[7])
    pack = B * (2 * n * iw * 4 * P + P * (mf + mg) * 4)
    fin = B * (P * (mf + mg) * 4 + (2 * n - 1) * ow * 4)
    return {"pack_bytes": pack, "finish_bytes": fin}


# -------------------------------------------------------------- multi-rank
def rank_env():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def max_over_ranks(x, dist=None, device=None):
    """Max of a host float over all ranks (timings are max over ranks)."""
    if dist is None:
        return x
    import torch
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def job_products(batch_per_rank, world):
    """Weak scaling: every rank multiplies its own batch of independent pairs."""
    return batch_per_rank * world


# ------------------------------------------------------------------ clocks
class ClockMonitor:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = os.path.join("/tmp", f"kmx_clocks_{os.getpid()}.csv")

    def start(self):
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=self.fh, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        self.proc.wait()
        self.fh.close()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        load = [s for s in sm if s > 500] or sm
        return {"sm_mhz": statistics.median(load) if load else None,
                "sm_max_mhz": max(mx) if mx else None, "samples": len(sm), "reasons": sorted(reasons)}


# ---------------------------------------------------------- GPU measurement
def run_ours(args, cfg, rank, world, local_rank):
    import numpy as np
    import torch

    import paper_0712_4046_b200 as kmx
    from paper_0712_4046_b200 import _lib

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    def mor(x):
        return max_over_ranks(x, dist, dev)

    fh, gh = make_inputs(cfg, rank)
    signed = cfg.get("signed", False)
    B = cfg["batch"]
    flush_buf = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream(dev)
    L = _lib.lib()
    peak = kmx.imad_peak(4096)  # live IMAD.WIDE.U32 microbenchmark, same process and clocks
    tpeak = kmx.tc_peak(2000)   # live dense tcgen05 u8 MMA microbenchmark (MAC/s)

    variants = [args.variant] + [v for v in (1, 2, 3, 4) if v != args.variant] if args.all_variants else [args.variant]
    per_variant = {}
    clocks = None
    headline = None
    for vi, v in enumerate(variants):
        if cfg["kind"] == "bks":
            op = kmx.BksBatch(v, B, cfg["lx"], cfg["ly"], cfg["b"], device=dev)
            fd = torch.from_numpy(fh).to(dev)
            gd = torch.from_numpy(gh).to(dev)
            out = torch.empty((B, 2 * cfg["lx"] - 1, 2 * cfg["ly"] - 1), dtype=torch.int64, device=dev)
        else:
            op = kmx.KsBatch(v, B, cfg["n"], cfg["n"], cfg["b"], signed=signed, device=dev)
            fd = torch.from_numpy(fh.view(np.int32)).to(dev)
            gd = torch.from_numpy(gh.view(np.int32)).to(dev)
            out = op.empty_out()
        for _ in range(args.warmup):
            op(fd, gd, out)
        op.status()
        graph = None
        if args.graphs:  # CUDA graph of the whole step (no per-kernel launch gaps)
            graph, out = op.capture(fd, gd, out)
            graph.replay()
            op.status()
        L.kmx_prof_enable(1)
        import ctypes
        prof = (ctypes.c_float * 6)()
        kern = [0.0] * 6
        mon = None
        if vi == 0 and rank == 0:
            mon = ClockMonitor(local_rank)
            mon.start()
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        total_ms = 0.0
        launches = 0
        for _ in range(args.steps):
            flush_buf.fill_(1)  # L2 flush between timed steps (untimed)
            e0.record(stream)
            if graph is not None:
                graph.replay()
            else:
                op(fd, gd, out)
            e1.record(stream)
            e1.synchronize()
            total_ms += e0.elapsed_time(e1)
            launches += L.kmx_last_launch_count()
            if graph is None:
                L.kmx_prof_read(prof, 6)
                for i in range(6):
                    kern[i] += prof[i]
        barrier()
        L.kmx_prof_enable(0)
        if mon is not None:
            clocks = mon.stop()
        op.status()
        if graph is not None:
            # per-kernel durations: CUDA events around each launch (kmx_prof),
            # eager launches right after the graph-timed region
            L.kmx_prof_enable(1)
            op(fd, gd, out)  # untimed: the unsplit shape's first call (plan autotuning)
            L.kmx_prof_read(prof, 6)
            for _ in range(args.steps):
                flush_buf.fill_(1)
                op(fd, gd, out)
                L.kmx_prof_read(prof, 6)
                for i in range(6):
                    kern[i] += prof[i]
            L.kmx_prof_enable(0)
        total_ms = mor(total_ms)
        ms = total_ms / args.steps
        rec = {"products_per_s": job_products(B, world) / (ms * 1e-3), "ms_per_step": ms, "launches_per_step": launches / args.steps}
        if cfg["kind"] == "bks":
            names = ["beval", "conv", "brecover"]
            rec["kernel_ms"] = {nm: kern[i] / args.steps for i, nm in enumerate(names) if kern[i] > 0}
            conv_ms = kern[1] / args.steps
            if conv_ms > 0:  # one IMAD.WIDE (int32 x int32 -> int64) per coefficient MAC
                rec["conv_macs_per_s"] = algorithmic_products(cfg, v) * B / (conv_ms * 1e-3)
                rec["conv_frac_of_imad_peak"] = rec["conv_macs_per_s"] / peak
        if cfg["kind"] == "ks":
            names = ["pack", "mul", "finish", "recon", "bias"]
            rec["kernel_ms"] = {nm: kern[i] / args.steps for i, nm in enumerate(names) if kern[i] > 0}
            if "recon" in rec["kernel_ms"] and "finish" not in rec["kernel_ms"]:  # K3 + K4 fused (k_finrec)
                rec["kernel_ms"]["finish+recon (fused)"] = rec["kernel_ms"].pop("recon")
            prods = algorithmic_products(cfg, v) * B
            mul_ms = kern[1] / args.steps
            rec["mul_limb_products_per_s"] = prods / (mul_ms * 1e-3) if mul_ms > 0 else None
            rec["mul_frac_of_imad_peak"] = rec["mul_limb_products_per_s"] / peak if mul_ms > 0 else None
            rec["mul_engine"] = kmx.mul_engine(v, cfg["n"], cfg["n"], cfg["b"], signed=signed)
            plan = (ctypes.c_int64 * 8)()
            if L.kmx_mul_plan(v, B, cfg["n"], cfg["n"], cfg["b"], _lib.KMX_SIGNED if signed else 0, plan) == 0:
                rec["mul_plan"] = {"engine": ["imad", "tensor tiled", "tensor chunked"][int(plan[0])],
                                   "H": int(plan[1]), "NW": int(plan[2]), "KC": int(plan[3]), "TPC": int(plan[4]),
                                   "mmas_per_product": int(plan[5]), "smem_bytes_per_product": int(plan[6]),
                                   "issued_byte_macs_per_product": int(plan[7])}
            if rec["mul_engine"] == "tensor" and mul_ms > 0:
                # algorithmic byte MACs of the u8 convolution: 16 per 32x32 limb product
                rec["mul_frac_of_tensor_peak"] = 16.0 * rec["mul_limb_products_per_s"] / tpeak
        per_variant[VNAME[v]] = rec
        if vi == 0:
            headline = (v, rec, op, fd, gd, out, launches)
        del op
    v, rec, op, fd, gd, out, launches = headline
    peaks = {"imad": peak, "tensor": tpeak}

    # ---- end to end through the public host API (pinned host buffers)
    e2e = None
    if cfg["kind"] == "ks":
        ow = L.kmx_ks_out_words(cfg["n"], cfg["n"], cfg["b"], _lib.KMX_SIGNED if signed else 0)
        fp = torch.from_numpy(fh.view(np.int32)).pin_memory().numpy().view(np.uint32)
        gp = torch.from_numpy(gh.view(np.int32)).pin_memory().numpy().view(np.uint32)
        hp = torch.empty((B, 2 * cfg["n"] - 1, ow), dtype=torch.int32).pin_memory().numpy().view(np.uint32)
        call = lambda: kmx.ks_mul_host(v, fp, gp, cfg["b"], signed=signed, out=hp)  # noqa: E731
        h2d = fp.nbytes + gp.nbytes
        d2h = hp.nbytes
    else:
        fp = torch.from_numpy(fh).pin_memory().numpy()
        gp = torch.from_numpy(gh).pin_memory().numpy()
        hp = torch.empty((B, 2 * cfg["lx"] - 1, 2 * cfg["ly"] - 1), dtype=torch.int64).pin_memory().numpy()
        call = lambda: kmx.bks_mul_host(v, fp, gp, cfg["b"], out=hp)  # noqa: E731
        h2d = fp.nbytes + gp.nbytes
        d2h = hp.nbytes
    for _ in range(max(1, args.warmup)):
        call()
    barrier()
    tot = 0.0
    for _ in range(args.steps):
        flush_buf.fill_(1)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        call()
        tot += time.perf_counter() - t0
    barrier()
    tot = mor(tot)
    e2e = {"value": job_products(B, world) / (tot / args.steps), "unit": "poly products/s",
           "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
           "ms_per_step": 1e3 * tot / args.steps, "api": "paper_0712_4046_b200.ks_mul_host -> kmx_ks_mul_host"
           if cfg["kind"] == "ks" else "paper_0712_4046_b200.bks_mul_host -> kmx_bks_mul_host"}

    # correctness spot check of the timed output against the oracle (pair 0)
    check = None
    if rank == 0:
        from oracle import ks_oracle as O
        from paper_0712_4046_b200.words import words_to_ints
        if cfg["kind"] == "ks":
            fi = to_ints(fh[:1], signed)[0]
            gi = to_ints(gh[:1], signed)[0]
            want = (O.ks_mul_signed(1, fi, gi, cfg["b"], mode="native") if signed
                    else O.ks_mul(1, fi, gi, cfg["b"], mode="native"))
            got = words_to_ints(out[0].cpu().numpy().view(np.uint32), signed=signed)
            check = got == want
        else:
            want = O.bks(v, fh[0].tolist(), gh[0].tolist())
            check = out[0].cpu().tolist() == want

    result = dict(rec=rec, per_variant=per_variant, e2e=e2e, peak=peak, tpeak=tpeak, clocks=clocks, variant=v,
                  launches=launches, check=check)
    if dist is not None:
        dist.destroy_process_group()
    return result


# ------------------------------------------------------------ CPU baseline
def _cpu_task(args):
    kind, v, f, g, b, signed = args
    from oracle import ks_oracle as O
    if kind == "bks":  # the reference's default UniMul (uni_schoolbook, oracle.py:58-69)
        return len(O.bks(v, f, g, umul=O.uni_schoolbook))
    if signed:
        return len(O.ks_mul_signed(v, f, g, b, mode="karatsuba"))
    return len(O.ks_mul(v, f, g, b, mode="karatsuba"))


def cpu_tasks(cfg, variant, count):
    fh, gh = make_inputs(cfg, 0)
    count = min(count, cfg["batch"])
    if cfg["kind"] == "bks":
        return [("bks", variant, fh[i].tolist(), gh[i].tolist(), cfg["b"], False) for i in range(count)]
    signed = cfg["signed"]
    fi = to_ints(fh[:count], signed)
    gi = to_ints(gh[:count], signed)
    return [("ks", variant, fi[i], gi[i], cfg["b"], signed) for i in range(count)]


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_baseline(cfg, variant, budget_s=12.0):
    """Oracle port of the reference algorithm (Python ints, restated
    Karatsuba as in bignat.py:344-371) over all host cores on a bounded
    sample of pairs of the same workload."""
    import multiprocessing as mp
    cores = host_cores()
    t0 = time.perf_counter()
    _cpu_task(cpu_tasks(cfg, variant, 1)[0])
    t_pair = max(1e-4, time.perf_counter() - t0)
    n = int(max(cores, min(cfg["batch"] * 4, budget_s * cores / t_pair)))
    if cfg["kind"] == "bks":
        n = cores  # one pair per core (seconds each through the pure-Python UniMul)
    tasks = cpu_tasks(cfg, variant, n)
    while len(tasks) < n:
        tasks += tasks[:n - len(tasks)]
    with mp.get_context("fork").Pool(cores) as pool:
        pool.map(_cpu_task, tasks[:cores])  # warm the workers
        t0 = time.perf_counter()
        pool.map(_cpu_task, tasks, chunksize=1)
        dt = time.perf_counter() - t0
    return {"value": len(tasks) / dt, "unit": "poly products/s", "cores": cores, "kind": "port",
            "sample": f"{len(tasks)} pairs of {cfg['desc']} through oracle/ks_oracle.py "
                      f"({VNAME[variant]}, restated reference Karatsuba on Python ints"
                      f"{', bias-lifted signed inputs' if cfg.get('signed') else ''}), "
                      f"multiprocessing over {cores} cores, {dt:.1f} s",
            "cpu_model": cpu_model()}


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def run_reference(args, cfg):
    import multiprocessing as mp
    cores = host_cores()
    v = args.variant
    per_step = cores * (1 if cfg["kind"] == "bks" else 2)  # bks: one pair per core per step
    tasks = cpu_tasks(cfg, v, per_step)
    while len(tasks) < per_step:
        tasks += tasks[:per_step - len(tasks)]
    times = []
    with mp.get_context("fork").Pool(cores) as pool:
        for _ in range(max(1, args.warmup)):
            pool.map(_cpu_task, tasks[:cores])
        for _ in range(args.steps):
            t0 = time.perf_counter()
            pool.map(_cpu_task, tasks, chunksize=1)
            times.append(time.perf_counter() - t0)
    ms = 1e3 * statistics.mean(times)
    value = per_step / (ms * 1e-3)
    return {
        "metric": METRIC, "value": value, "unit": "poly products/s", "impl": "reference",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int (Python)",
        "data": "synthetic (seeded numpy PCG64, BASELINE shapes)",
        "config": config_json(cfg, v),
        "cpu_baseline": {"value": value, "unit": "poly products/s", "cores": cores, "kind": "port",
                         "sample": f"{per_step} pairs per step of {cfg['desc']} ({VNAME[v]}) through "
                                   f"oracle/ks_oracle.py over {cores} cores (the reference is pure "
                                   f"Python; its restatement runs here because /root/reference is "
                                   f"absent on the GPU box)", "cpu_model": cpu_model()},
        "e2e": {"value": value, "unit": "poly products/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def config_json(cfg, v):
    c = {"workload": f"{cfg['desc']}, variant {VNAME[v]} ({VDESC[v]})", "variant": VNAME[v],
         "variant_naming": "reference kronmul names: ks2 = reciprocal, ks3 = negated",
         "batch": cfg["batch"], "coeff_bits": cfg["b"],
         "l2": "flushed between timed steps (256 MiB device write, untimed)"}
    if cfg["kind"] == "ks":
        c.update({"n": cfg["n"], "signed": cfg["signed"]})
    else:
        c.update({"lx": cfg["lx"], "ly": cfg["ly"]})
    return c


def load_traffic(config_name, variant, key="mul_dram_bytes"):
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        d = json.load(open(path))
        return d[config_name][VNAME[variant]][key]
    except Exception:
        return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--variant", type=int, default=4, choices=[1, 2, 3, 4])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-all-variants", dest="all_variants", action="store_false")
    ap.add_argument("--no-cpu-baseline", dest="cpu_baseline", action="store_false")
    ap.add_argument("--no-graphs", dest="graphs", action="store_false",
                    help="launch kernels eagerly instead of replaying a captured CUDA graph")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    cfg = CONFIGS[args.config]
    rank, world, local_rank = rank_env()

    if args.impl == "reference":
        if rank == 0:
            print(json.dumps(run_reference(args, cfg)), flush=True)
        return

    r = run_ours(args, cfg, rank, world, local_rank)
    if rank != 0:
        return
    v = r["variant"]
    rec = r["rec"]
    line = {
        "metric": METRIC, "value": rec["products_per_s"], "unit": "poly products/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": rec["ms_per_step"],
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32 limbs (exact integer)",
        "data": "synthetic (seeded numpy PCG64, BASELINE shapes)", "config": config_json(cfg, v),
        "parallelism": f"replicas x{world} (independent pairs, no collective)",
        "cuda_graph": bool(args.graphs),
    }
    if cfg["kind"] == "ks":
        mul_ms = rec["kernel_ms"].get("mul")
        prods = algorithmic_products(cfg, v) * cfg["batch"]
        ach = prods / (mul_ms * 1e-3) / 1e9
        imad_view = {"bound": "imad", "kernel": "k_mul (IMAD.WIDE.U32 schoolbook)",
                     "achieved": ach, "peak": r["peak"] / 1e9, "unit": "G limb-products/s",
                     "frac": ach * 1e9 / r["peak"],
                     "peak_source": "kmx_imad_peak() microbenchmark measured live in this process",
                     "algorithmic_work": f"{prods} 32x32->64 limb products per launch "
                                         f"({algorithmic_products(cfg, v)} per pair x {cfg['batch']})"}
        if rec.get("mul_engine") == "tensor":
            tops = 2.0 * 16.0 * prods / (mul_ms * 1e-3) / 1e12
            tpk = 2.0 * r["tpeak"] / 1e12
            line["roofline"] = {
                "bound": "tensor", "kernel": "k_tcmul (tcgen05.mma kind::i8 byte convolution, TMEM s32)",
                "achieved": tops, "peak": tpk, "unit": "TOPS (int8, 2 ops per MAC)", "frac": tops / tpk,
                "peak_source": "kmx_tc_peak() live: dense tcgen05 u8 MMA M=128 N=256 K=32 from smem, all SMs",
                "algorithmic_work": f"{16 * prods} byte MACs per launch (16 per 32x32 limb product; "
                                    f"{algorithmic_products(cfg, v)} limb products per pair x {cfg['batch']})",
                "traffic": load_traffic(args.config, v, "tcmul_dram_bytes"),
                "same_kernel_in_imad_units": {"achieved": ach, "unit": "G limb-products/s",
                                              "frac_of_imad_peak": ach * 1e9 / r["peak"]}}
            mp_ = rec.get("mul_plan")
            if mp_ and mp_["engine"] == "tensor tiled" and mp_["smem_bytes_per_product"]:
                # what bounds it: the SS-mode MMAs read A (128 x 32 B) and B (16H x 32 B)
                # from shared memory per MMA; peak = 128 B/clk/SM at the observed SM clock
                P_ = {1: 1, 2: 2, 3: 2, 4: 4}[v]
                nprod = cfg["batch"] * P_
                clk = (r["clocks"] or {}).get("sm_mhz") or 1965.0
                smem_peak = 148 * 128 * clk * 1e6 / 1e9
                smem_ach = mp_["smem_bytes_per_product"] * nprod / (mul_ms * 1e-3) / 1e9
                line["roofline"]["smem_operand_bound"] = {
                    "achieved": smem_ach, "peak": smem_peak, "unit": "GB/s", "frac": smem_ach / smem_peak,
                    "bytes_per_launch": mp_["smem_bytes_per_product"] * nprod,
                    "plan": {k: mp_[k] for k in ("H", "NW", "KC", "TPC", "mmas_per_product")},
                    "algorithmic_fraction_of_issued_macs": 16.0 * algorithmic_products(cfg, v) / P_ /
                    mp_["issued_byte_macs_per_product"] if mp_["issued_byte_macs_per_product"] else None,
                    "note": "peak = 148 SMs x 128 B/clk shared-memory bandwidth at the observed SM clock"}
        else:
            imad_view["traffic"] = load_traffic(args.config, v)
            line["roofline"] = imad_view
        pu = pack_unpack_bytes(cfg, v)
        try:
            peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
            hbm = peaks["hbm_gbs"]
            src = "MEASURED_PEAKS.json hbm_gbs"
        except Exception:
            hbm, src = 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"
        km = rec["kernel_ms"]
        fin_ms = km.get("finish", km.get("finish+recon (fused)"))
        line["roofline_hbm"] = {"bound": "hbm", "unit": "GB/s", "peak": hbm, "peak_source": src,
                                "finish": {"achieved": pu["finish_bytes"] / (fin_ms * 1e-3) / 1e9,
                                           "frac": pu["finish_bytes"] / (fin_ms * 1e-3) / 1e9 / hbm,
                                           "kernel": "k_finrec (finish + reconstruct fused)"
                                           if "finish" not in km else "k_finish_w / k_finish"}}
        if "pack" in km:
            line["roofline_hbm"]["pack"] = {"achieved": pu["pack_bytes"] / (km["pack"] * 1e-3) / 1e9,
                                            "frac": pu["pack_bytes"] / (km["pack"] * 1e-3) / 1e9 / hbm}
        else:
            line["roofline_hbm"]["pack"] = "fused into the tensor-core multiply (operands packed in shared memory)"
    else:
        macs = algorithmic_products(cfg, v) * cfg["batch"]
        cms = rec["kernel_ms"].get("conv")
        ach = macs / (cms * 1e-3) / 1e9 if cms else None
        line["roofline"] = {"bound": "imad", "kernel": "k_conv (int32 x int32 -> int64 IMAD.WIDE convolution)",
                            "achieved": ach, "peak": r["peak"] / 1e9, "unit": "G MAC/s",
                            "frac": ach * 1e9 / r["peak"] if ach else None,
                            "peak_source": "kmx_imad_peak() microbenchmark measured live in this process",
                            "algorithmic_work": f"{macs} coefficient MACs per launch "
                                                f"({algorithmic_products(cfg, v)} per pair x {cfg['batch']})",
                            "traffic": load_traffic(args.config, v, "conv_dram_bytes")}
    pv = r["per_variant"]
    line["per_variant"] = pv
    if all(VNAME[x] in pv for x in (1, 2, 3, 4)):
        base = pv["ks1"]["products_per_s"]
        line["speed_ratios_vs_ks1"] = {k: pv[k]["products_per_s"] / base for k in ("ks1", "ks2", "ks3", "ks4")}
    line["e2e"] = r["e2e"]
    line["gpu_launches"] = int(r["launches"])
    line["clocks"] = r["clocks"]
    line["oracle_spot_check_pair0"] = r["check"]
    if world == 1 and args.cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(cfg, v)
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
