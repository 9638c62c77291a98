#!/usr/bin/env python
"""Benchmark of the B200 Cubical Ripser hot path (one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5b] [--impl ours|reference]

Workload.  BASELINE.json's metric names no config, so the headline is the largest workload:
configs[4]'s batch C5b -- 64 volumes of 128^3 (Gaussian random field, sigma = 3, +inf outside a
centred ball of radius 60), full barcode H0-H2.  Batches are independent problems, so at N GPUs
the job is N such batches, one per rank (rank 0: the config's own batch, seed 6; rank r > 0: the
same recipe from seed (6, r)), with no exchange during compute: weak scaling, `scaling` "weak",
value = all ranks' voxels / the max-over-ranks time.  A step is one full barcode computation of
every rank's batch: every SURVEY §8(a) row runs (filtration + apparent pairs, H0 union-find, the
dimension-1 coboundary reduction, the top dimension by duality, output), then (N > 1) the bars
are gathered onto rank 0.  The same run also times configs[4]'s single 384^3 volume (C5) on rank 0 at N = 1
(key "c5_single").  Other configs (--config c1..c5, c2f64) remain available as parity cases.

Timing: W >= 3 untimed warm-up steps; then K steps bracketed by CUDA events on the launching
stream; barrier + synchronize on both sides of the timed region; max over ranks.  The C5b input
(537 MB) exceeds L2 (126 MB), so no flush is needed; for configs whose input fits in L2 a
256 MiB write flushes it before every step (outside the events).  ``e2e`` repeats the
measurement through the host-buffer entry points (cr_barcodes_batched_host / cr_barcodes_host)
with pinned buffers: H2D of the inputs and D2H of bars + offsets inside the timed region, and at
N > 1 the gather of every shard's bars onto rank 0's host.
``--impl reference`` times the CPU oracle (oracle/, test infrastructure) on a bounded sample,
without importing the product package.
"""
from __future__ import annotations

import argparse
import json
import os
import resource
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "voxels/sec full barcode (dims 0..d), HBM GB/s vs peak; bit-exact vs oracle"
CONFIG_DESC = {
    "c1": "2D 128x128 iid U[0,1) float32, H0+H1",
    "c2": "1D Gaussian random walk, 2^24 float32 samples, H0",
    "c3": "65536 x 28x28 blob images (0..255 levels), H0+H1 (one such batch per rank)",
    "c4": "3D 128^3 GRF sigma=2, H0-H2",
    "c5": "3D 384^3 GRF sigma=3, +inf outside ball r=180, H0-H2",
    "c5b": "64 x 128^3 GRF sigma=3, +inf outside ball r=60, H0-H2 (one such batch per rank)",
    "c2f64": "1D Gaussian random walk, 2^24 float64 samples (kept in double), H0",
}
F64 = {"c2f64"}
BATCHED = {"c3", "c5b"}
L2_BYTES = 126 * 2 ** 20


def shard_range(n: int, rank: int, world: int):
    """Contiguous, balanced slice [start, stop) of n items (same rule as the package's dist.py;
    repeated here so that the reference arm never imports the product)."""
    base, extra = divmod(n, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy burst)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled every 200 ms during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,utilization.gpu,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.lines = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.t = threading.Thread(target=self._read, daemon=True)
        self.t.start()
        t0 = time.time()
        while not self.lines and time.time() - t0 < 5:
            time.sleep(0.02)

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        rows = []
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                rows.append((float(parts[0]), float(parts[1]), float(parts[2]), parts[3:7]))
            except ValueError:
                continue
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        loaded = [r for r in rows if r[2] > 0] or rows
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i, v in enumerate(r[3]) if v.lower() == "active"})
        return {"sm_mhz": float(np.median([r[0] for r in loaded])), "sm_max_mhz": rows[0][1],
                "reasons": reasons, "samples": len(rows), "samples_under_load": len(loaded)}


def c5b_volumes(k: int = 64, rank: int = 0):
    """The first k volumes of the C5b batch (the generator draws them in sequence); rank r > 0 of
    a multi-GPU job draws its own batch from seed (6, r)."""
    from workloads import generators as gen
    g = np.random.default_rng(6 if rank == 0 else (6, rank))
    return np.stack([gen.masked_grf((128, 128, 128), 3.0, 60.0, g) for _ in range(k)]), 2


def make_input(cfg: str, rank: int, world: int):
    """(this rank's input, maxdim, units in the whole job).  Batches: one whole batch per rank
    (weak scaling, see the module docstring)."""
    from workloads import generators as gen
    if cfg == "c3":
        imgs = gen.blobs(65536, 3 if rank == 0 else (3, rank))
        return imgs, 1, len(imgs) * world
    if cfg == "c5b":
        vols, md = c5b_volumes(64, rank)
        return vols, md, len(vols) * world
    if cfg == "c2f64":
        return gen.random_walk(1 << 24, 2, dtype=np.float64), 0, 1
    img, md = gen.config(cfg)
    return img, md, 1


def khalimsky_cells(shape):
    n = 1
    for v in shape:
        n *= 2 * int(v) - 1
    return n


def stacked_shape(shape, batch):
    """The batched general path stacks the images along their slowest axis with one +inf
    separator layer between consecutive images (R16)."""
    return (batch * (int(shape[0]) + 1) - 1,) + tuple(int(v) for v in shape[1:])


def algorithmic_bytes(stage, nvox, kcells, n_out, K=0, D=3):
    """Bytes a stage must move once."""
    if stage == "1d_level1":
        return 4 * nvox + 8 * n_out               # read the series, stage (birth, death) per bar
    if stage == "1d_levels_gather":
        return 20 * n_out                         # read staged pairs, write 12-B output bars
    if stage in ("f64_rank", "f64_cast"):        # read the doubles, write the float32 surrogate
        return 12 * nvox + (8 * nvox if stage == "f64_rank" else 0)
    if stage == "f64_map":
        return 12 * n_out + 24 * n_out
    if stage == "filtration":
        # K1+K2 fused: read the image, write births + tags, the H0 basin forest and (D >= 2) the
        # top-dimension dual forest (4 B per voxel each), and list the residual present edges
        # (and, 3D, squares) -- 4 B each, K of them
        return 4 * nvox + 5 * kcells + 4 * nvox + (4 * nvox if D >= 2 else 0) + 4 * K
    return None


NCU_KERNEL = {"1d_level1": "k1_level1", "1d_levels_gather": "k1_levels_coop",
              "filtration": "k_filtration", "reduce_d1": "k_reduce"}


def ncu_summary(kernel, config):
    """The committed ncu --set full summary (profiles/rNN/sM/ncu_full_<config>_summary.json) of
    `kernel` for this config from the newest round and session (numeric order), or {}."""
    import glob
    import re

    def key(p):
        m = re.search(r"profiles/r(\d+)/s(\d+)/", p.replace(os.sep, "/"))
        return (int(m.group(1)), int(m.group(2))) if m else (-1, -1)
    paths = glob.glob(os.path.join(ROOT, "profiles", "r*", "s*", f"ncu_full_{config}_summary.json"))
    for p in sorted(paths, key=key, reverse=True):
        try:
            with open(p) as f:
                ks = json.load(f)["kernels"]
            # template instances are summarised as name<args> (k_filtration<0>: the product's
            # cp.async ring)
            name = kernel if kernel in ks else next(k for k in ks if k.split("<")[0] == kernel)
            return dict(ks[name], source=os.path.relpath(p, ROOT), kernel_instance=name)
        except (KeyError, OSError, ValueError, StopIteration):
            continue
    return {}


def host_info():
    info = {"cpu_model": None, "nproc": os.cpu_count(), "ram_gb": None}
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                info["cpu_model"] = ln.split(":", 1)[1].strip()
                break
        for ln in open("/proc/meminfo"):
            if ln.startswith("MemTotal"):
                info["ram_gb"] = round(int(ln.split()[1]) / 2 ** 20, 1)
                break
    except OSError:
        pass
    return info


def _oracle_one(args):
    """Worker: the oracle on one image; returns (seconds, peak RSS of this worker in GB)."""
    import oracle
    img, md = args
    t0 = time.perf_counter()
    oracle.ph(img, md, dtype=img.dtype)
    dt = time.perf_counter() - t0
    return dt, resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 2 ** 20


def oracle_pool(images, md, procs):
    """The oracle, as it stands, over `images` in a pool of `procs` worker processes.
    Returns (wall seconds, max worker peak RSS GB)."""
    from multiprocessing import get_context
    import oracle
    oracle.build()
    ctx = get_context("fork")
    t0 = time.perf_counter()
    with ctx.Pool(procs) as pool:
        res = pool.map(_oracle_one, [(im, md) for im in images], chunksize=1)
    return time.perf_counter() - t0, max(r[1] for r in res)


def cpu_baseline(cfg, host_img, maxdim):
    """The oracle (single-threaded C++, oracle/), as it stands, on a bounded sample of the
    workload: one unit on one core, and (batched configs) a pool of P = min(nproc, 64) processes
    over P units; value = the pool's voxels/s, cores = P."""
    import oracle
    oracle.build()
    hi = host_info()
    if cfg in BATCHED:
        one = host_img[0]
        dt1, rss1 = oracle_pool([one], maxdim, 1)  # one worker process: its own peak RSS
        P = max(1, min(os.cpu_count() or 1, 64, len(host_img)))
        sample = host_img[:P] if len(host_img) >= P else host_img
        wall, rss = oracle_pool(list(sample), maxdim, P)
        nv = float(np.prod(sample.shape))
        return {"value": nv / wall, "unit": "voxels/s", "cores": P, "kind": "oracle",
                "sample": f"{len(sample)} {cfg} units, one per worker process (pool of {P})",
                "seconds": round(wall, 2),
                "single_core": {"value": float(np.prod(one.shape)) / dt1, "unit": "voxels/s",
                                "sample": f"1 {cfg} unit", "seconds": round(dt1, 2),
                                "peak_rss_gb": round(rss1, 2)},
                "peak_rss_gb_per_worker": round(rss, 2), **hi}
    if cfg in ("c2", "c2f64", "c1", "c4"):
        sample, desc = host_img, f"full {cfg}, one run"
    else:  # c5: the central 192^3 crop keeps the sample bounded (~20 s)
        sample, desc = host_img[96:288, 96:288, 96:288], "central 192^3 crop of C5"
    dt, rss = _oracle_one((np.ascontiguousarray(sample), maxdim))
    return {"value": float(np.prod(sample.shape)) / dt, "unit": "voxels/s", "cores": 1,
            "kind": "oracle", "sample": desc, "seconds": round(dt, 2),
            "peak_rss_gb": round(rss, 2), **hi}


def run_ours(args, rank, world, local_rank):
    import ctypes
    import torch
    import torch.distributed as dist
    import paper_2005_12692_b200 as cr
    from paper_2005_12692_b200.dist import gather_barcodes

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    host_img, maxdim, units_total = make_input(args.config, rank, world)
    batched = args.config in BATCHED
    f64 = args.config in F64
    nvox_local = int(np.prod(host_img.shape))
    img = torch.from_numpy(np.ascontiguousarray(host_img)).to(dev)
    stream = torch.cuda.current_stream(dev)
    gloo = dist.new_group(backend="gloo") if world > 1 else None

    if batched:
        shape = tuple(img.shape[1:])
        nb = int(img.shape[0])
        cap = max(cr.max_pairs(shape, maxdim) * nb, 1)
        kshape = stacked_shape(shape, nb)
        nvox_dev, kcells = int(np.prod(kshape)), khalimsky_cells(kshape)
    else:
        shape = tuple(img.shape)
        cap = cr.max_pairs(shape, maxdim)
        nvox_dev, kcells = nvox_local, khalimsky_cells(shape)
    pairs = torch.empty((cap, 3), dtype=torch.int32, device=dev)
    offsets = torch.empty((img.shape[0] + 1,), dtype=torch.int64, device=dev) if batched else None

    def step(src=None):
        if batched:
            n = ctypes.c_int64(0)
            src = img if src is None else src
            st = cr._lib.cr_barcodes_batched(src.data_ptr(), nb, cr._shape(shape), len(shape),
                                             maxdim, pairs.data_ptr(), None, cap,
                                             offsets.data_ptr(), ctypes.byref(n),
                                             ctypes.c_void_p(stream.cuda_stream))
            cr._check(st)
            m = int(n.value)
            if world > 1:  # the job ends with every shard's barcodes on rank 0, in input order
                got = gather_barcodes(pairs[:m], offsets)
                return int(got[0].shape[0]) if got is not None else m
            return m
        if f64:
            return len(cr.barcodes_f64(img, maxdim, capacity=cap).dim)
        return len(cr.barcodes(img, maxdim, out=(pairs, None)).pairs)

    small_input = nvox_local * host_img.itemsize <= L2_BYTES
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev) if small_input else None
    cr.set_profiling(True)
    for _ in range(args.warmup):
        n_out = step()
    torch.cuda.synchronize()
    stats_warm = cr.last_stats()

    sampler = ClockSampler(local_rank) if rank == 0 else None
    if dist.is_initialized():
        dist.barrier()
    torch.cuda.synchronize()
    if sampler:
        sampler.start()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    stage_tot, launches, k5 = {}, 0, {"additions": 0, "addlen": 0}
    for k in range(args.steps):
        if flush is not None:
            flush.zero_()
        ev[k][0].record(stream)
        n_out = step()
        ev[k][1].record(stream)
        st = cr.last_stats()
        launches += st["launches"]
        k5["additions"] += st["additions"][1]
        k5["addlen"] += st["addlen"][1]
        for name, ms in st["stages"].items():
            stage_tot[name] = stage_tot.get(name, 0.0) + ms
    torch.cuda.synchronize()
    if dist.is_initialized():
        dist.barrier()
    torch.cuda.synchronize()
    clocks = sampler.stop() if sampler else None
    times = [a.elapsed_time(b) for a, b in ev]
    total_ms = sum(times)
    if dist.is_initialized():
        t = torch.tensor([total_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    if batched:
        nvox_total = int(np.prod(host_img.shape[1:])) * units_total
    else:
        nvox_total = nvox_local * world
    value = nvox_total / (ms_per_step / 1e3)

    # ---- end to end through the host entry points (pinned buffers, copies inside the region)
    e2e = None
    if batched:
        pin_in = torch.from_numpy(np.ascontiguousarray(host_img)).pin_memory()
        pin_pairs = torch.empty((cap, 3), dtype=torch.int32).pin_memory()
        pin_off = torch.empty((nb + 1,), dtype=torch.int64).pin_memory()
        d2h = {"bytes": 0}

        def e2e_step():
            bc, off = cr.barcodes_batched_host(pin_in, maxdim, out=(pin_pairs, pin_off, None),
                                               stream=stream)
            m = int(off[-1])
            d2h["bytes"] = m * 12 + (nb + 1) * 8
            if world > 1:  # every shard's bars onto rank 0's host (gloo over the host copies)
                got = gather_barcodes(pin_pairs[:m], pin_off, group=gloo)
                return int(got[0].shape[0]) if got is not None else m
            return m
        h2d = nvox_local * 4
    elif f64:
        pin_in = torch.from_numpy(np.ascontiguousarray(host_img)).pin_memory()
        dev_in = torch.empty_like(pin_in, device=dev)
        d2h = {"bytes": 0}

        def e2e_step():
            dev_in.copy_(pin_in, non_blocking=True)
            bc = cr.barcodes_f64(dev_in, maxdim, capacity=cap)
            res = (bc.dim.cpu(), bc.birth.cpu(), bc.death.cpu())
            d2h["bytes"] = len(res[0]) * 20
            return len(res[0])
        h2d = nvox_local * 8
    else:
        pin_in = torch.from_numpy(np.ascontiguousarray(host_img)).pin_memory()
        pin_out = torch.empty((cap, 3), dtype=torch.int32).pin_memory()
        d2h = {"bytes": 0}

        def e2e_step():
            bc = cr.barcodes_host(pin_in, maxdim, out=(pin_out, None), stream=stream)
            d2h["bytes"] = len(bc.pairs) * 12
            return len(bc.pairs)
        h2d = nvox_local * 4
    for _ in range(max(1, min(args.warmup, 2))):
        e2e_step()
    torch.cuda.synchronize()
    if dist.is_initialized():
        dist.barrier()
    e2e_ev = []
    for k in range(args.steps):
        if flush is not None:
            flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        e2e_step()
        b.record(stream)
        e2e_ev.append((a, b))
    torch.cuda.synchronize()
    e2e_ms = sum(a.elapsed_time(b) for a, b in e2e_ev)
    if dist.is_initialized():
        t = torch.tensor([e2e_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e = {"value": nvox_total / (e2e_ms / args.steps / 1e3), "unit": "voxels/s",
           "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h["bytes"],
           "ms_per_step": e2e_ms / args.steps,
           "api": ("cr_barcodes_batched_host" if batched else
                   "cr_barcodes_f64 (+ torch copies)" if f64 else "cr_barcodes_host")}

    # ---- configs[4]'s single 384^3 volume, timed in the same run (rank 0, N = 1)
    c5_single = None
    if batched and args.config == "c5b" and world == 1 and not args.no_c5:
        from workloads import generators as gen
        v5, md5 = gen.config("c5")
        t5 = torch.from_numpy(v5).to(dev)
        cap5 = cr.max_pairs(v5.shape, md5)
        out5 = (torch.empty((cap5, 3), dtype=torch.int32, device=dev), None)
        cr.barcodes(t5, md5, out=out5)
        ts, st5 = [], None
        for _ in range(args.c5_steps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            n5 = len(cr.barcodes(t5, md5, out=out5).pairs)
            b.record(stream)
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
            st5 = cr.last_stats()
        ms5 = float(np.median(ts))
        c5_single = {"workload": "c5: " + CONFIG_DESC["c5"], "ms_per_call_median": round(ms5, 3),
                     "ms_per_call": [round(x, 3) for x in ts],
                     "voxels_per_s": v5.size / (ms5 / 1e3),
                     "in_domain_voxels_per_s": float(np.isfinite(v5).sum()) / (ms5 / 1e3),
                     "bars": n5, "stages_ms": {k: round(v, 4) for k, v in st5["stages"].items()},
                     "k5_dim1": {"columns": st5["columns"][1], "additions": st5["additions"][1],
                                 "entry_work": st5["addlen"][1]}}
        del t5

    if rank != 0:
        return None
    hbm, peak_src = peaks()
    st = stats_warm
    stage_avg = {k: v / args.steps for k, v in stage_tot.items()}
    dom = max(stage_avg, key=stage_avg.get) if stage_avg else None
    # roofline: the filtration + apparent-pair kernel (k_filtration, K1+K2 fused) against HBM --
    # the kernel north_star's bandwidth target names; 1D configs: the dominant 1D kernel
    roof_stage = "filtration" if "filtration" in stage_avg else dom
    roof = None
    listed, D = 0, sum(1 for n in (kshape if batched else shape) if n > 1)
    if st and st.get("cells") and st.get("apparent"):
        c, a = st["cells"], st["apparent"]
        listed = max(c[1] - a[0] - a[1], 0) + (max(c[2] - a[1] - a[2], 0) if D == 3 else 0)
    alg = (algorithmic_bytes(roof_stage, nvox_dev, kcells, n_out, K=listed, D=D)
           if roof_stage else None)
    if alg:
        ach = alg / (stage_avg[roof_stage] / 1e3) / 1e9
        ncu = ncu_summary(NCU_KERNEL.get(roof_stage, ""), args.config)
        traffic = None
        if ncu.get("dram_read_MB") is not None:
            traffic = round((ncu["dram_read_MB"] + ncu["dram_write_MB"]) * 1e6)
        roof = {"bound": "hbm", "kernel": NCU_KERNEL.get(roof_stage, roof_stage),
                "achieved": round(ach, 1), "peak": hbm, "unit": "GB/s",
                "frac": round(ach / hbm, 4), "traffic": traffic,
                "alg_bytes_per_launch": alg, "avg_ms": round(stage_avg[roof_stage], 5),
                "share_of_step": round(stage_avg[roof_stage] / ms_per_step, 4),
                "peak_source": peak_src, "traffic_source": ncu.get("source")}
        if ncu.get("warp_instructions"):
            # what bounds the kernel as built: instruction issue (4 schedulers x SMs x clock),
            # its warp instructions from the same ncu capture, timed live like `achieved`
            sms = torch.cuda.get_device_properties(0).multi_processor_count
            mhz = (clocks or {}).get("sm_mhz") or (clocks or {}).get("sm_max_mhz") or 1965.0
            ipeak = 4 * sms * mhz * 1e6 / 1e9
            iach = ncu["warp_instructions"] / (stage_avg[roof_stage] / 1e3) / 1e9
            roof["issue"] = {"warp_instructions": ncu["warp_instructions"],
                             "achieved": round(iach, 1), "peak": round(ipeak, 1),
                             "unit": "G warp-instructions/s", "frac": round(iach / ipeak, 4),
                             "alu_pipe_pct_ncu": ncu.get("alu_pipe_pct"),
                             "note": "ALU-issue bound as built (DESIGN.md §6 K1+K2 fused)"}
    # the dominant stage (the dims >= 1 reduction for 3D): latency-bound, reported as throughput
    dominant = None
    if dom:
        dominant = {"stage": dom, "kernel": NCU_KERNEL.get(dom, dom), "avg_ms": round(stage_avg[dom], 4),
                    "share_of_step": round(stage_avg[dom] / ms_per_step, 4)}
        if dom == "reduce_d1" and k5["additions"]:
            secs = stage_tot[dom] / 1e3
            entry_gbs = k5["addlen"] * 8 / secs / 1e9
            dominant.update({"bound": "latency (dependent column additions, DESIGN.md §6)",
                             "additions_per_s": k5["additions"] / secs,
                             "entry_bytes_per_s_GB": round(entry_gbs, 2),
                             "entry_bytes_frac_of_hbm": round(entry_gbs / hbm, 5)})
    out = {
        "metric": METRIC, "value": value, "unit": "voxels/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64" if f64 else "f32",
        "data": "synthetic (seeded, workloads/generators.py)",
        "config": {"workload": f"{args.config}: {CONFIG_DESC[args.config]}",
                   "voxels_per_step": nvox_total, "maxdim": maxdim,
                   "parallelism": (f"dp{world} (one batch per rank, gather to rank 0)" if batched
                                   else f"replicas x{world} (one image per rank)"),
                   "l2": ("flushed before every timed step (256 MiB write, outside the events)"
                          if flush is not None else
                          f"input ({nvox_local * host_img.itemsize / 2**20:.0f} MiB per rank) "
                          "larger than L2 (126 MiB): no flush"),
                   "bars_per_step": n_out},
        "ms_per_step_all": [round(x, 3) for x in times],
        "roofline": roof,
        "dominant_stage": dominant,
        "stages_ms": {k: round(v, 5) for k, v in stage_avg.items()},
        "clocks": clocks,
        "e2e": e2e,
        "gpu_launches": launches,
        "stats": {k: st[k] for k in ("cells", "apparent", "columns", "rounds", "pairs", "path",
                                     "additions", "maxlen")},
    }
    if c5_single:
        out["c5_single"] = c5_single
    if world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(args.config, host_img, maxdim)
    return out


def run_reference(args, rank, world):
    """--impl reference: the CPU oracle timed on the host cores, rank 0 only; each step is a
    bounded sample of the workload (batched configs: P = min(nproc, 64) units in a pool of P
    worker processes).  Never imports the product package."""
    if rank != 0:
        return None
    import oracle
    oracle.build()
    if args.config == "c5b":
        P = max(1, min(os.cpu_count() or 1, 64))
        host_img, maxdim = c5b_volumes(min(P, 64))
    else:
        host_img, maxdim, _ = make_input(args.config, 0, 1)
        P = max(1, min(os.cpu_count() or 1, 64, len(host_img))) if args.config in BATCHED else 1
    if args.config in ("c2", "c2f64"):
        sample, desc = host_img[: 1 << 20], f"first 2^20 samples of {args.config} per step, 1 core"
    elif args.config in BATCHED:
        sample = host_img[:P]
        desc = f"{len(sample)} {args.config} units per step, one per worker (pool of {P})"
    elif args.config == "c5":
        sample, desc = host_img[160:224, 160:224, 160:224], "central 64^3 crop of C5 per step, 1 core"
    else:
        sample, desc = host_img, f"full {args.config} per step, 1 core"

    def one():
        if args.config in BATCHED:
            return oracle_pool(list(sample), maxdim, P)[0]
        t0 = time.perf_counter()
        oracle.ph(sample, maxdim, dtype=sample.dtype)
        return time.perf_counter() - t0

    for _ in range(args.warmup):
        one()
    dt = sum(one() for _ in range(args.steps)) / args.steps
    v = float(np.prod(sample.shape)) / dt
    cores = P if args.config in BATCHED else 1
    return {"impl": "reference", "metric": METRIC, "value": v, "unit": "voxels/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3,
            "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64" if args.config in F64 else "f32",
            "data": "synthetic (seeded, workloads/generators.py)",
            "config": {"workload": f"{args.config}: {CONFIG_DESC[args.config]}", "maxdim": maxdim},
            "cpu_baseline": {"value": v, "unit": "voxels/s", "cores": cores, "kind": "oracle",
                             "sample": desc, **host_info()},
            "e2e": {"value": v, "unit": "voxels/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c5b", choices=sorted(CONFIG_DESC))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-c5", action="store_true", help="skip the C5 single-volume timing")
    ap.add_argument("--c5-steps", type=int, default=3)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        out = run_reference(args, rank, world)
    else:
        import torch
        import torch.distributed as dist
        if world > 1:
            torch.cuda.set_device(local_rank)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        out = run_ours(args, rank, world, local_rank)
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
    if out is not None:
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
