#!/usr/bin/env python
"""Benchmark of the multipoint Kronecker-substitution hot path on B200.

Metric (BASELINE.json): polynomial products per second per KS variant, with
the multiply kernel's fraction of its measured peak (dense tcgen05 u8 MMA rate
on the tensor cores, IMAD.WIDE.U32 rate on the integer pipe) and the HBM
fractions of the pack / finish / reconstruction kernels.

Headline workload = BASELINE config 2 (configs[1]): Z[x], signed int32
coefficients, batch 1024 pairs, n = 1024, variant ks4.  A step = one pass of
the hot path (pack -> multiply -> finish [-> reconstruct]) over the whole
batch.  The default single-GPU run also measures every other BASELINE config
under the same clock and prints them inside the same JSON line:
``per_config`` (c1, c3, c4: all four variants, kernel split, rooflines, e2e,
parity) and ``c5`` (the 30-point crossover sweep, all four variants, parity
per point).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c1|c2|c3|c4]
                  [--variant 1..4] [--impl ours|reference] [--quick]

One JSON line on rank 0.  ``--gpus N`` (N > 1) without a torchrun
environment relaunches itself under torch.distributed.run with N ranks; every
rank multiplies its own batch (independent pairs, no collective on the data
path: weak scaling) and the step time is the max over ranks.
``--impl reference`` times the reference algorithm's CPU implementation (the
oracle port of kronmul, 0-16% slower per pair than the reference itself,
profiles/r02/port_vs_reference.json) on all host cores of rank 0.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import math
import os
import socket
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "poly products/sec per KS variant; fraction of the tensor (or IMAD) peak and HBM roofline"
VNAME = {1: "ks1", 2: "ks2", 3: "ks3", 4: "ks4"}
VDESC = {1: "standard 2^N", 2: "reciprocal 2^N,2^-N", 3: "negated +-2^N", 4: "four-point +-2^N,+-2^-N"}
PCOUNT = {1: 1, 2: 2, 3: 2, 4: 4}
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
C5_NS = (16, 64, 256, 1024, 4096, 8192)
C5_BITS = (8, 32, 64, 128, 256)
L2_FLUSH_BYTES = 256 << 20


def c5_config(n, b, scale=1):
    B = int(math.ceil(1e6 / (2 * n - 1))) * scale
    return dict(kind="ks", batch=B, n=n, b=b, signed=False, seed=5000 + 17 * n + b,
                desc=f"c5: Z[x] u{b}, batch {B}, n={n}")


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


# ------------------------------------------------------------ work / bytes
def ks_geometry(cfg, variant):
    """Derived sizes of one pair (kmx_ks_params, ksint.py:82-98): the variant
    actually run (KS4 -> KS1 fallback), P, operand limbs, digit streams."""
    from paper_0712_4046_b200 import _lib
    p = (ctypes.c_int64 * 8)()
    flags = _lib.KMX_SIGNED if cfg["signed"] else 0
    n, b = cfg["n"], cfg["b"]
    _lib.check(_lib.lib().kmx_ks_params(variant, n, n, b, flags, p))
    e, N1, N2, N4, safe, k = (int(p[i]) for i in range(6))
    v = variant
    if v == 4 and (not safe or k == 1):
        v = 1
    ne, no = (k + 1) // 2, k // 2
    if v == 2:  # fwd/rev, k+1 digits of N2 bits
        streams = [(k + 1, N2)] * 2
    elif v == 4:  # fwd/rev even and odd, n_even+1 / n_odd+1 digits of 2 N4 bits
        streams = [(ne + 1, 2 * N4), (no + 1, 2 * N4)] * 2
    else:
        streams = []
    ow = _lib.lib().kmx_ks_out_words(n, n, b, flags)
    return dict(variant=v, P=PCOUNT[v], mf=int(p[6]), mg=int(p[7]), streams=streams, out_words=ow,
                in_words=1 if cfg["signed"] else (b + 31) // 32, k=k)


def algorithmic_products(cfg, variant):
    """Schoolbook 32x32 limb products per pair: sum over the
    sub-products of m_f * m_g, m = ceil((N (L-1) + b + 2) / 32) limbs; for the
    bivariate config the coefficient MACs of the univariate products."""
    if cfg["kind"] == "bks":
        lx, ly = cfg["lx"], cfg["ly"]
        Lu = {1: (2 * lx - 1) * (ly - 1) + lx, 2: lx * ly, 3: lx * ly, 4: (lx + 1) // 2 * (ly - 1) + lx}[variant]
        return PCOUNT[variant] * Lu * Lu
    g = ks_geometry(cfg, variant)
    return g["P"] * g["mf"] * g["mg"]


def hbm_bytes(cfg, variant):
    """Algorithmic HBM bytes per step of the kernels around the multiply:
    pack reads the inputs once and writes the packed operands; finish reads
    the products and writes the coefficients (ks1/ks3) or the digit streams
    (ks2/ks4); reconstruction reads the digit streams and writes the
    coefficients."""
    if cfg["kind"] == "bks":
        return None
    g = ks_geometry(cfg, variant)
    B, n = cfg["batch"], cfg["n"]
    inputs = 2 * n * g["in_words"] * 4
    operands = g["P"] * (g["mf"] + g["mg"]) * 4
    coeffs = g["k"] * g["out_words"] * 4
    digits = sum(cnt * ((w + 31) // 32) * 4 for cnt, w in g["streams"])
    out = {"pack": B * (inputs + operands),
           "finish": B * (operands + (digits if g["streams"] else coeffs))}
    if g["streams"]:
        out["recon"] = B * (digits + coeffs)
        out["fused"] = B * (operands + coeffs)  # k_finrec: the digit streams stay on chip
    return out


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


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def relaunch_under_torchrun(n):
    """``--gpus N`` outside torchrun: run N ranks (one per GPU) under
    torch.distributed.run on this node; rank 0 prints the line."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), os.path.abspath(__file__),
           *sys.argv[1:]]
    return subprocess.call(cmd)


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
class Gpu:
    """Per-process measurement context: device, L2 flush buffer, live peaks."""

    def __init__(self, local_rank, dist=None):
        import torch

        import paper_0712_4046_b200 as kmx
        from paper_0712_4046_b200 import _lib
        self.torch, self.kmx, self._lib = torch, kmx, _lib
        self.dev = torch.device("cuda", local_rank)
        torch.cuda.set_device(self.dev)
        self.dist = dist
        self.L = _lib.lib()
        self.flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.int32, device=self.dev)
        self.stream = torch.cuda.current_stream(self.dev)
        self.imad = kmx.imad_peak(4096)  # live IMAD.WIDE.U32 microbenchmark (limb products/s)
        self.tensor = kmx.tc_peak(2000)  # live dense tcgen05 u8 MMA microbenchmark (MAC/s)
        self._shape_peaks = {}
        try:
            self.hbm = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
            self.hbm_src = "MEASURED_PEAKS.json hbm_gbs"
        except Exception:
            self.hbm, self.hbm_src = 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"

    def tc_shape_peak(self, n):
        """Dense SS-mode u8 MMA rate at M=128 and this N (kmx_tc_peak_n): the
        ceiling of K2's own tile shape, where every MMA re-reads its A tile."""
        if n not in self._shape_peaks:
            self._shape_peaks[n] = float(self.L.kmx_tc_peak_n(n, 2000))
        return self._shape_peaks[n]

    def barrier(self):
        if self.dist is not None:
            self.dist.barrier()
        self.torch.cuda.synchronize()

    def mor(self, x):
        return max_over_ranks(x, self.dist, self.dev)

    def traffic(self, cfg_name, variant, key):
        """Per-launch DRAM bytes of a kernel from the committed ncu capture
        (profiles/ncu_traffic.json, captured at the commit it names)."""
        try:
            d = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
            return d["configs"][cfg_name][VNAME[variant]][key]
        except Exception:
            return None


def _op_for(g, cfg, v):
    torch, kmx = g.torch, g.kmx
    if cfg["kind"] == "bks":
        op = kmx.BksBatch(v, cfg["batch"], cfg["lx"], cfg["ly"], cfg["b"], device=g.dev)
        out = torch.empty((cfg["batch"], 2 * cfg["lx"] - 1, 2 * cfg["ly"] - 1), dtype=torch.int64, device=g.dev)
    else:
        op = kmx.KsBatch(v, cfg["batch"], cfg["n"], cfg["n"], cfg["b"], signed=cfg.get("signed", False),
                         device=g.dev)
        out = op.empty_out()
    return op, out


KS_SLOTS = ["pack", "mul", "finish", "recon", "bias"]
BKS_SLOTS = ["beval", "conv", "brecover"]


def kernel_split(g, op, fd, gd, out, steps):
    """Per-kernel durations: CUDA events recorded on the launch stream around
    each launch (kmx_prof_*), eager calls with the L2 flushed before each."""
    prof = (ctypes.c_float * 6)()
    kern = [0.0] * 6
    g.L.kmx_prof_enable(1)
    op(fd, gd, out)  # untimed: the unsplit shape's first call (plan autotuning)
    g.L.kmx_prof_read(prof, 6)
    for _ in range(steps):
        g.flush.fill_(1)
        op(fd, gd, out)
        g.L.kmx_prof_read(prof, 6)
        for i in range(6):
            kern[i] += prof[i]
    g.L.kmx_prof_enable(0)
    return [k / steps for k in kern]


def measure_variant(g, cfg, cfg_name, v, fd, gd, steps, warmup, graphs=True, monitor=None):
    """Device-timed products/s of one variant (CUDA-graph replay, L2 flushed
    between timed steps, CUDA events on the launch stream, max over ranks),
    plus the per-kernel split and the rooflines.  Returns (record, output)."""
    torch = g.torch
    op, out = _op_for(g, cfg, v)
    for _ in range(warmup):
        op(fd, gd, out)
    op.status()
    graph = None
    if graphs:
        graph, out = op.capture(fd, gd, out)
        graph.replay()
        op.status()
    launches = g.L.kmx_last_launch_count()
    if monitor is not None:
        monitor.start()
    g.barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    total_ms = 0.0
    for _ in range(steps):
        g.flush.fill_(1)  # L2 flush between timed steps (untimed)
        e0.record(g.stream)
        if graph is not None:
            graph.replay()
        else:
            op(fd, gd, out)
        e1.record(g.stream)
        e1.synchronize()
        total_ms += e0.elapsed_time(e1)
    g.barrier()
    clocks = monitor.stop() if monitor is not None else None
    op.status()
    kern = kernel_split(g, op, fd, gd, out, steps)
    op.status()
    world = 1 if g.dist is None else g.dist.get_world_size()
    ms = g.mor(total_ms) / steps
    B = cfg["batch"]
    rec = {"products_per_s": job_products(B, world) / (ms * 1e-3), "ms_per_step": ms,
           "gpu_launches_per_step": launches}
    if cfg["kind"] == "bks":
        rec["kernel_ms"] = {nm: kern[i] for i, nm in enumerate(BKS_SLOTS) if kern[i] > 0}
        conv_ms = kern[1]
        macs = algorithmic_products(cfg, v) * B
        ach = macs / (conv_ms * 1e-3) if conv_ms > 0 else None
        uni = int(g.L.kmx_bks_uni_engine(v, cfg["lx"], cfg["ly"], cfg["b"]))
        if uni > 0:
            # univariate products on the integer KS path (pack -> tcgen05 multiply
            # -> finish [-> reconstruct]); its MAC rate beside the integer pipe's peak
            rec["roofline"] = {"bound": "tensor", "kernel": f"univariate products through the integer KS path "
                                                            f"(ks{uni}: pack, k_tcmul, finish, reconstruct)",
                               "achieved": ach / 1e9 if ach else None, "unit": "G coefficient-MAC/s",
                               "frac": None, "frac_of_imad_peak": ach / g.imad if ach else None,
                               "peak_source": "work-equivalent: the IMAD.WIDE convolution would be bound by "
                                              "kmx_imad_peak(); the KS path runs on the tensor cores",
                               "algorithmic_work": f"{macs} coefficient MACs per launch "
                                                   f"({algorithmic_products(cfg, v)} per pair x {B})"}
        else:
            rec["roofline"] = {"bound": "imad", "kernel": "k_conv (int32 x int32 -> int64 IMAD.WIDE convolution)",
                               "achieved": ach / 1e9 if ach else None, "peak": g.imad / 1e9, "unit": "G MAC/s",
                               "frac": ach / g.imad if ach else None,
                               "peak_source": "kmx_imad_peak() microbenchmark measured live in this process",
                               "algorithmic_work": f"{macs} coefficient MACs per launch "
                                                   f"({algorithmic_products(cfg, v)} per pair x {B})",
                               "traffic": g.traffic(cfg_name, v, "conv_dram_bytes")}
    else:
        km = {nm: kern[i] for i, nm in enumerate(KS_SLOTS) if kern[i] > 0}
        if "recon" in km and "finish" not in km:  # K3 + K4 fused (k_finrec)
            km["finish+recon (fused)"] = km.pop("recon")
        rec["kernel_ms"] = km
        rec["roofline"] = mul_roofline(g, cfg, cfg_name, v, km.get("mul"), clocks)
        rec["roofline_hbm"] = hbm_roofline(g, cfg, v, km)
    if clocks is not None:
        rec["clocks"] = clocks
    return rec, out, op


def mul_roofline(g, cfg, cfg_name, v, mul_ms, clocks):
    """K2's roofline: the tcgen05 byte convolution against the live dense u8
    MMA peak, or the integer-pipe schoolbook against the live IMAD peak."""
    from paper_0712_4046_b200 import _lib
    if not mul_ms:
        return None
    B = cfg["batch"]
    prods = algorithmic_products(cfg, v) * B
    lps = prods / (mul_ms * 1e-3)
    flags = _lib.KMX_SIGNED if cfg["signed"] else 0
    plan = (ctypes.c_int64 * 8)()
    eng = g.kmx.mul_engine(v, cfg["n"], cfg["n"], cfg["b"], signed=cfg["signed"])
    karatsuba = None
    info = {}
    if g.L.kmx_mul_plan(v, B, cfg["n"], cfg["n"], cfg["b"], flags, plan) == 0:
        info = {"engine": ["imad", "tensor tiled", "tensor chunked", "karatsuba",
                           "tensor swizzled-window", "tensor swizzled-window M=64"][min(5, int(plan[0]))],
                "H": int(plan[1]), "NW": int(plan[2]), "KC": int(plan[3]), "TPC": int(plan[4]),
                "mmas_per_product": int(plan[5]), "smem_bytes_per_product": int(plan[6]),
                "issued_byte_macs_per_product": int(plan[7])}
    if hasattr(g.L, "kmx_mul_karatsuba_levels"):
        karatsuba = int(g.L.kmx_mul_karatsuba_levels(v, B, cfg["n"], cfg["n"], cfg["b"], flags))
    work = (f"{prods} 32x32->64 limb products per launch ({algorithmic_products(cfg, v)} per pair x {B}; "
            f"schoolbook count, the work the reference's classical multiply does)")
    if eng == "tensor":
        tops = 2.0 * 16.0 * lps / 1e12
        tpk = 2.0 * g.tensor / 1e12
        kname = ("k_tcswz (tcgen05.mma kind::i8 byte convolution: swizzled sliding windows x phase table, TMEM s32)"
                 if str(info.get("engine", "")).startswith("tensor swizzled-window")
                 else "k_tcmul (tcgen05.mma kind::i8 byte convolution, TMEM s32)")
        r = {"bound": "tensor", "kernel": kname,
             "achieved": tops, "peak": tpk, "unit": "TOPS (int8, 2 ops per MAC)", "frac": tops / tpk,
             "peak_source": "kmx_tc_peak() live: dense tcgen05 u8 MMA M=128 N=256 K=32 from smem, all SMs",
             "algorithmic_work": f"{16 * prods} byte MACs per launch (16 per 32x32 limb product); " + work,
             "traffic": g.traffic(cfg_name, v, "tcmul_dram_bytes"),
             "same_kernel_in_imad_units": {"achieved": lps / 1e9, "unit": "G limb-products/s",
                                           "frac_of_imad_peak": lps / g.imad}}
        m64 = info.get("engine") == "tensor swizzled-window M=64"
        if info.get("engine") in ("tensor tiled", "tensor swizzled-window", "tensor swizzled-window M=64") and info.get("H"):
            n_mma = 16 * info["H"]
            sp = g.tc_shape_peak(n_mma)
            nprod_ = B * PCOUNT[ks_geometry(cfg, v)["variant"]]
            issued = info["issued_byte_macs_per_product"] * nprod_ / (mul_ms * 1e-3) if info.get(
                "issued_byte_macs_per_product") else None
            r["same_shape_ceiling"] = {
                "mma_shape": (f"M=64 N={n_mma} K=32 issued (two 64-row windows); ceiling measured at M=128 N={n_mma}"
                              if m64 else f"M=128 N={n_mma} K=32 (SS, u8)"), "peak": 2.0 * sp / 1e12, "unit": "TOPS",
                "frac_algorithmic": 2.0 * 16.0 * lps / (2.0 * sp) if sp > 0 else None,
                "frac_issued": issued / sp if (issued and sp > 0) else None,
                "note": "kmx_tc_peak_n(): the dense rate of the MMA shape K2 issues; frac_issued counts every MAC "
                        "the tiles issue (incl. the Toeplitz zero padding), frac_algorithmic only the product's"}
        if info.get("engine") in ("tensor tiled", "tensor swizzled-window", "tensor swizzled-window M=64") and info.get(
                "smem_bytes_per_product"):
            nprod = B * PCOUNT[ks_geometry(cfg, v)["variant"]]
            clk = (clocks or {}).get("sm_mhz") or 1965.0
            smem_peak = 148 * 128 * clk * 1e6 / 1e9
            smem_ach = info["smem_bytes_per_product"] * nprod / (mul_ms * 1e-3) / 1e9
            r["smem_operand_bound"] = {
                "achieved": smem_ach, "peak": smem_peak, "unit": "GB/s", "frac": smem_ach / smem_peak,
                "bytes_per_launch": info["smem_bytes_per_product"] * nprod,
                "plan": {k: info[k] for k in ("H", "NW", "KC", "TPC", "mmas_per_product")},
                "algorithmic_fraction_of_issued_macs": (16.0 * prods / nprod / info["issued_byte_macs_per_product"]
                                                        if info["issued_byte_macs_per_product"] else None),
                "note": "peak = 148 SMs x 128 B/clk shared-memory bandwidth at the observed SM clock"}
    else:
        r = {"bound": "imad", "kernel": "k_mul (IMAD.WIDE.U32 schoolbook)",
             "achieved": lps / 1e9, "peak": g.imad / 1e9, "unit": "G limb-products/s", "frac": lps / g.imad,
             "peak_source": "kmx_imad_peak() microbenchmark measured live in this process",
             "algorithmic_work": work, "traffic": g.traffic(cfg_name, v, "mul_dram_bytes")}
    r["mul_plan"] = info
    if karatsuba:
        r["karatsuba_levels"] = karatsuba
    return r


def hbm_roofline(g, cfg, v, km):
    """Algorithmic bytes / CUDA-event duration of pack, finish and
    reconstruction against the measured HBM bandwidth."""
    by = hbm_bytes(cfg, v)
    out = {"bound": "hbm", "unit": "GB/s", "peak": g.hbm, "peak_source": g.hbm_src,
           "bytes_per_step": by}

    def ent(name, nbytes, ms, kernel):
        if not ms or not nbytes:
            return None
        a = nbytes / (ms * 1e-3) / 1e9
        return {"achieved": a, "frac": a / g.hbm, "bytes": nbytes, "ms": ms, "kernel": kernel}

    out["pack"] = ent("pack", by["pack"], km.get("pack"), "k_pack_pair / k_pack")
    if "finish+recon (fused)" in km:
        out["finish+recon"] = ent("finish+recon", by["fused"], km["finish+recon (fused)"], "k_finrec")
    else:
        out["finish"] = ent("finish", by["finish"], km.get("finish"), "k_finish_w / k_finish / k_finchunk")
        if "recon" in by:
            out["recon"] = ent("recon", by["recon"], km.get("recon"), "k_recon_pair / k_recon_cl / k_recon_par")
    return out


def measure_e2e(g, cfg, v, fh, gh, steps, warmup, dev_out):
    """End to end through the public host API (pinned host buffers; H2D copy
    of the inputs, the kernels and the D2H copy of the result inside the
    timed call), and a full-batch comparison with the device-path output."""
    import numpy as np
    torch, kmx = g.torch, g.kmx
    if cfg["kind"] == "ks":
        signed = cfg["signed"]
        ow = dev_out.shape[2]
        fp = torch.from_numpy(fh.view(np.int32)).pin_memory().numpy().view(np.uint32)
        gp = torch.from_numpy(gh.view(np.int32)).pin_memory().numpy().view(np.uint32)
        hp = torch.empty((cfg["batch"], 2 * cfg["n"] - 1, ow), dtype=torch.int32).pin_memory().numpy().view(np.uint32)
        call = lambda: kmx.ks_mul_host(v, fp, gp, cfg["b"], signed=signed, out=hp)  # noqa: E731
        api = "paper_0712_4046_b200.ks_mul_host -> kmx_ks_mul_host"
    else:
        fp = torch.from_numpy(fh).pin_memory().numpy()
        gp = torch.from_numpy(gh).pin_memory().numpy()
        hp = torch.empty((cfg["batch"], 2 * cfg["lx"] - 1, 2 * cfg["ly"] - 1), dtype=torch.int64).pin_memory().numpy()
        call = lambda: kmx.bks_mul_host(v, fp, gp, cfg["b"], out=hp)  # noqa: E731
        api = "paper_0712_4046_b200.bks_mul_host -> kmx_bks_mul_host"
    for _ in range(max(1, warmup)):
        call()
    g.barrier()
    tot = 0.0
    for _ in range(steps):
        g.flush.fill_(1)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        call()
        tot += time.perf_counter() - t0
    g.barrier()
    tot = g.mor(tot)
    world = 1 if g.dist is None else g.dist.get_world_size()
    same = bool(np.array_equal(hp.view(np.uint8), dev_out.cpu().numpy().view(np.uint8)))
    return {"value": job_products(cfg["batch"], world) / (tot / steps), "unit": "poly products/s",
            "h2d_bytes_per_step": int(fp.nbytes + gp.nbytes), "d2h_bytes_per_step": int(hp.nbytes),
            "ms_per_step": 1e3 * tot / steps, "api": api, "equals_device_output": same}


def oracle_pairs(cfg, B):
    """Pairs checked against the oracle: the first and last of every part a
    batch split (2 or 4 parts) or the host path's chunking can produce, i.e.
    0, B/4, B/2, 3B/4 and their predecessors, and B-1."""
    cand = {0, B - 1}
    for q in (4, 2):
        for i in range(1, q):
            s = (B * i) // q
            cand.update({s, s - 1})
    return sorted(p for p in cand if 0 <= p < B)


def check_pairs(cfg, v, fh, gh, out, pairs):
    import numpy as np
    from oracle import ks_oracle as O
    from paper_0712_4046_b200.words import words_to_ints
    host = out.cpu().numpy()
    ok = True
    for p in pairs:
        if cfg["kind"] == "bks":
            ok = ok and host[p].tolist() == O.bks(v, fh[p].tolist(), gh[p].tolist())
            continue
        signed = cfg["signed"]
        fi = to_ints(fh[p:p + 1], signed)[0]
        gi = to_ints(gh[p:p + 1], signed)[0]
        want = (O.ks_mul_signed(1, fi, gi, cfg["b"], mode="native") if signed
                else O.ks_mul(1, fi, gi, cfg["b"], mode="native"))
        ok = ok and words_to_ints(host[p].view(np.uint32), signed=signed) == want
    return bool(ok)


def measure_config(g, cfg_name, cfg, variants, steps, warmup, graphs=True, e2e=True, monitor_first=False,
                   rank=0, oracle=True, pairs=None):
    """Every variant of one config; parity: all variants bit-identical on
    the whole batch, and the oracle on pairs from every split part."""
    torch = g.torch
    import numpy as np
    fh, gh = make_inputs(cfg, rank)
    if cfg["kind"] == "bks":
        fd, gd = torch.from_numpy(fh).to(g.dev), torch.from_numpy(gh).to(g.dev)
    else:
        fd = torch.from_numpy(fh.view(np.int32)).to(g.dev)
        gd = torch.from_numpy(gh.view(np.int32)).to(g.dev)
    recs, outs = {}, {}
    for i, v in enumerate(variants):
        mon = ClockMonitor(g.dev.index) if (monitor_first and i == 0 and rank == 0) else None
        rec, out, op = measure_variant(g, cfg, cfg_name, v, fd, gd, steps, warmup, graphs, mon)
        if e2e:
            rec["e2e"] = measure_e2e(g, cfg, v, fh, gh, max(3, steps // 2), 1, out)
        recs[VNAME[v]] = rec
        outs[v] = out.clone()
        del op
    res = {"workload": cfg["desc"], "batch": cfg["batch"], "variants": recs}
    base = recs.get("ks1")
    if base:
        res["speed_ratios_vs_ks1"] = {k: r["products_per_s"] / base["products_per_s"] for k, r in recs.items()}
    ref = outs[variants[0]]
    par = {"variants_bit_identical_full_batch": all(torch.equal(ref, o) for o in outs.values())}
    if oracle and rank == 0:
        pairs = pairs if pairs is not None else oracle_pairs(cfg, cfg["batch"])
        par["oracle_pairs"] = pairs
        par["oracle_ok"] = check_pairs(cfg, variants[0], fh, gh, ref, pairs)
    if e2e:
        par["e2e_equals_device_all_variants"] = all(r["e2e"]["equals_device_output"] for r in recs.values())
    res["parity"] = par
    return res


def c5_summary(g, steps, warmup, scale=1, ns=C5_NS, bits=C5_BITS, detail=False):
    """BASELINE config 5: the crossover sweep, all four variants per point;
    parity per point: the four variants bit-identical on the whole batch and
    the oracle on the first and last pair."""
    points = []
    t0 = time.time()
    for n in ns:
        for b in bits:
            cfg = c5_config(n, b, scale)
            res = measure_config(g, "c5", cfg, [4, 1, 2, 3], steps, warmup, e2e=False,
                                 pairs=[0, cfg["batch"] - 1])
            pt = {"n": n, "bits": b, "batch": cfg["batch"]}
            for k in ("ks1", "ks2", "ks3", "ks4"):
                pt[k] = res["variants"][k]["products_per_s"]
            pt["fastest"] = max(res["variants"], key=lambda k: res["variants"][k]["products_per_s"])
            pt["parity_ok"] = bool(res["parity"]["variants_bit_identical_full_batch"] and res["parity"]["oracle_ok"])
            if detail:
                pt["detail"] = res["variants"]
            else:
                pt["mul_frac"] = {k: (r["roofline"] or {}).get("frac") for k, r in res["variants"].items()}
                pt["mul_engine"] = {k: (r["roofline"] or {}).get("bound") for k, r in res["variants"].items()}
                pt["hbm_frac"] = {k: {s: (r["roofline_hbm"].get(s) or {}).get("frac")
                                      for s in ("pack", "finish", "recon", "finish+recon") if r["roofline_hbm"].get(s)}
                                  for k, r in res["variants"].items()}
            points.append(pt)
    return {"config": "BASELINE configs[4]: n x bits crossover sweep over Z[x], unsigned uniform from seed, "
                      "B = ceil(1e6/(2n-1)) pairs per point",
            "scale": scale, "steps": steps, "points": points, "wall_s": time.time() - t0,
            "all_parity_ok": all(p["parity_ok"] for p in points)}


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
    count = max(1, min(count, cfg["batch"]))
    if cfg["kind"] == "bks":
        tasks = [("bks", variant, fh[i].tolist(), gh[i].tolist(), cfg["b"], False) for i in range(count)]
    else:
        signed = cfg["signed"]
        fi = to_ints(fh[:count], signed)
        gi = to_ints(gh[:count], signed)
        tasks = [("ks", variant, fi[i], gi[i], cfg["b"], signed) for i in range(count)]
    return tasks


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def cpu_rate_1core(cfg, v, budget_s):
    """Serial, in this process: pairs/s of the oracle port on one core."""
    tasks = cpu_tasks(cfg, v, 64)
    _cpu_task(tasks[0])
    n, t0 = 0, time.perf_counter()
    while True:
        _cpu_task(tasks[n % len(tasks)])
        n += 1
        dt = time.perf_counter() - t0
        if dt >= budget_s or n >= 4 * cfg["batch"]:
            return n / dt, n, dt


def cpu_rate_all(cfg, v, cores, budget_s, pool):
    t0 = time.perf_counter()
    _cpu_task(cpu_tasks(cfg, v, 1)[0])
    t_pair = max(1e-4, time.perf_counter() - t0)
    n = int(max(cores, min(cfg["batch"] * 4, budget_s * cores / t_pair)))
    if cfg["kind"] == "bks":
        n = cores  # one pair per core (seconds each through the pure-Python UniMul)
    tasks = cpu_tasks(cfg, v, n)
    while len(tasks) < n:
        tasks += tasks[:n - len(tasks)]
    pool.map(_cpu_task, tasks[:cores])  # warm the workers
    t0 = time.perf_counter()
    pool.map(_cpu_task, tasks, chunksize=1)
    dt = time.perf_counter() - t0
    return len(tasks) / dt, len(tasks), dt


def cpu_baseline(cfg, variants, headline, budget_all=4.0, budget_1=2.0, one_core=True):
    """The oracle port of the reference algorithm (Python ints, restated
    reference Karatsuba, bignat.py:344-371) on the host cores, on a bounded
    sample of pairs of the same workload: all cores (multiprocessing over
    pairs, as the reference's README recommends) and one core, per variant."""
    import multiprocessing as mp
    cores = host_cores()
    per = {}
    with mp.get_context("fork").Pool(cores) as pool:
        for v in variants:
            r_all, n_all, dt_all = cpu_rate_all(cfg, v, cores, budget_all, pool)
            e = {"all_cores": r_all, "all_cores_sample": f"{n_all} pairs in {dt_all:.1f} s"}
            if one_core and cfg["kind"] == "ks":
                r1, n1, dt1 = cpu_rate_1core(cfg, v, budget_1)
                e["one_core"] = r1
                e["one_core_sample"] = f"{n1} pairs in {dt1:.1f} s"
            per[VNAME[v]] = e
    h = per[VNAME[headline]]
    return {"value": h["all_cores"], "unit": "poly products/s", "cores": cores, "kind": "port",
            "one_core_value": h.get("one_core"),
            "sample": f"{h['all_cores_sample']} of {cfg['desc']} through oracle/ks_oracle.py "
                      f"({VNAME[headline]}, restated reference Karatsuba on Python ints"
                      f"{', bias-lifted signed inputs' if cfg.get('signed') else ''}), "
                      f"multiprocessing over {cores} cores",
            "per_variant": per, "cpu_model": cpu_model()}


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
                                   f"absent on the GPU box; measured 0-16% slower per pair than the reference's "
                                   f"own (profiles/r02/port_vs_reference.json), so a GPU/port ratio overstates the GPU/reference ratio by at most that)",
                         "cpu_model": cpu_model()},
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--variant", type=int, default=4, choices=[1, 2, 3, 4])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--quick", action="store_true",
                    help="headline config and variant only (no per_config / c5 / CPU baseline)")
    ap.add_argument("--no-all-variants", dest="all_variants", action="store_false")
    ap.add_argument("--no-cpu-baseline", dest="cpu_baseline", action="store_false")
    ap.add_argument("--no-per-config", dest="per_config", action="store_false")
    ap.add_argument("--no-c5", dest="c5", action="store_false")
    ap.add_argument("--no-graphs", dest="graphs", action="store_false",
                    help="launch kernels eagerly instead of replaying a captured CUDA graph")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    if args.quick:
        args.all_variants = args.cpu_baseline = args.per_config = args.c5 = False
    cfg = CONFIGS[args.config]
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(relaunch_under_torchrun(args.gpus))
    rank, world, local_rank = rank_env()
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")

    if args.impl == "reference":
        if rank == 0:
            print(json.dumps(run_reference(args, cfg)), flush=True)
        return

    import torch
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    g = Gpu(local_rank, dist)
    v = args.variant
    variants = [v] + [x for x in (1, 2, 3, 4) if x != v] if args.all_variants else [v]
    head = measure_config(g, args.config, cfg, variants, args.steps, args.warmup, args.graphs,
                          e2e=True, monitor_first=True, rank=rank)
    rec = head["variants"][VNAME[v]]
    per_config, c5 = {}, None
    if world == 1 and args.per_config:
        for name in ("c1", "c2", "c3", "c4"):
            if name != args.config:
                per_config[name] = measure_config(g, name, CONFIGS[name], [1, 2, 3, 4], args.steps,
                                                  args.warmup, args.graphs, e2e=True)
    if world == 1 and args.c5:
        c5 = c5_summary(g, max(3, args.steps // 4), 3)
    if dist is not None:
        dist.destroy_process_group()
    if rank != 0:
        return
    line = {
        "metric": METRIC, "value": rec["products_per_s"], "unit": "poly products/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": rec["ms_per_step"],
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32 limbs (exact integer)",
        "data": "synthetic (seeded numpy PCG64, BASELINE shapes)", "config": config_json(cfg, v),
        "parallelism": f"replicas x{world} (independent pairs, no collective)",
        "cuda_graph": bool(args.graphs),
        "roofline": rec["roofline"],
    }
    if "roofline_hbm" in rec:
        line["roofline_hbm"] = rec["roofline_hbm"]
    line["kernel_ms"] = rec["kernel_ms"]
    line["per_variant"] = head["variants"]
    if "speed_ratios_vs_ks1" in head:
        line["speed_ratios_vs_ks1"] = head["speed_ratios_vs_ks1"]
    line["parity"] = head["parity"]
    line["e2e"] = rec["e2e"]
    line["gpu_launches"] = int(rec["gpu_launches_per_step"]) * args.steps
    line["gpu_launches_per_step"] = int(rec["gpu_launches_per_step"])
    line["clocks"] = rec.get("clocks")
    line["peaks"] = {"imad_limb_products_per_s": g.imad, "tensor_u8_macs_per_s": g.tensor, "hbm_gbs": g.hbm}
    if per_config:
        line["per_config"] = per_config
    if c5 is not None:
        line["c5"] = c5
    if world == 1 and args.cpu_baseline:
        cb = cpu_baseline(cfg, variants, v)
        for k, e in cb["per_variant"].items():
            gpu = head["variants"][k]
            e["gpu_over_all_cores"] = gpu["products_per_s"] / e["all_cores"]
            e["e2e_over_all_cores"] = gpu["e2e"]["value"] / e["all_cores"]
            if e.get("one_core"):
                e["gpu_over_one_core"] = gpu["products_per_s"] / e["one_core"]
        line["cpu_baseline"] = cb
        if per_config:
            for name, pc in per_config.items():
                c = CONFIGS[name]
                pcb = cpu_baseline(c, [1, 2, 3, 4], 4, budget_all=2.0, one_core=False)
                for k, e in pcb["per_variant"].items():
                    e["gpu_over_all_cores"] = pc["variants"][k]["products_per_s"] / e["all_cores"]
                pc["cpu_baseline"] = {"cores": pcb["cores"], "kind": "port", "per_variant": pcb["per_variant"]}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
