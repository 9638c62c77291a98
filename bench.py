#!/usr/bin/env python
"""Benchmark of the B200 Cubical Ripser hot path (one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]

A step is one full barcode computation (all SURVEY §8(a) rows the config exercises) over one
batch of seeded synthetic input already resident in HBM.  The default workload is BASELINE.json
configs[1] (C2: 1D Gaussian random walk of 2^24 float32 samples, H0) -- the config BASELINE's
metric is quoted on; configs[0] (C1) is the small parity case.

Timing: W untimed warm-up steps; then K steps, each bracketed by CUDA events on the launching
stream, with an L2 flush (a 256 MiB write, outside the events) before every step because the C2
input (64 MiB) is smaller than L2; barrier + synchronize on both sides of the timed region;
max over ranks.  Multi-GPU: one process per GPU (torchrun); single-image configs run one
independent replica per rank (weak scaling, no collective), batched configs (c3, c5b) are sharded
image-by-image across ranks.  ``e2e`` repeats the measurement through cr_barcodes_host with
pinned host buffers (host->device input copy and device->host bar copy inside the timed region).
``--impl reference`` times the CPU oracle (oracle/, test infrastructure) on a bounded sample.
"""
from __future__ import annotations

import argparse
import json
import os
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
    "c3": "65536 x 28x28 blob images (0..255 levels), H0+H1, sharded by image",
    "c4": "3D 128^3 GRF sigma=2, H0-H2",
    "c5": "3D 384^3 GRF sigma=3, +inf outside ball r=180, H0-H2",
    "c5b": "64 x 128^3 GRF sigma=3 in ball r=60, H0-H2, sharded by volume",
    "c2f64": "1D Gaussian random walk, 2^24 float64 samples (kept in double), H0",
}
F64 = {"c2f64"}
BATCHED = {"c3", "c5b"}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
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


def make_input(cfg: str, rank: int, world: int):
    from workloads import generators as gen
    from paper_2005_12692_b200.dist import shard_range
    if cfg == "c3":
        imgs = gen.blobs(65536, 3)
        a, b = shard_range(len(imgs), rank, world)
        return imgs[a:b], 1, len(imgs)
    if cfg == "c5b":
        vols, md = gen.config("c5b")
        a, b = shard_range(len(vols), rank, world)
        return vols[a:b], md, len(vols)
    if cfg == "c2f64":
        return gen.random_walk(1 << 24, 2, dtype=np.float64), 0, 1
    img, md = gen.config(cfg)
    return img, md, 1


def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    import paper_2005_12692_b200 as cr

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    host_img, maxdim, units_total = make_input(args.config, rank, world)
    batched = args.config in BATCHED
    f64 = args.config in F64
    nvox_local = int(np.prod(host_img.shape))
    img = torch.from_numpy(np.ascontiguousarray(host_img)).to(dev)
    stream = torch.cuda.current_stream(dev)

    if batched:
        shape = tuple(img.shape[1:])
        cap = cr.max_pairs(shape, maxdim) * int(img.shape[0])
    else:
        shape = tuple(img.shape)
        cap = cr.max_pairs(shape, maxdim)
    pairs = torch.empty((cap, 3), dtype=torch.int32, device=dev)
    offsets = torch.empty((img.shape[0] + 1,), dtype=torch.int64, device=dev) if batched else None

    def step(src=None):
        if batched:
            import ctypes
            n = ctypes.c_int64(0)
            src = img if src is None else src
            st = cr._lib.cr_barcodes_batched(src.data_ptr(), int(img.shape[0]), cr._shape(shape),
                                             len(shape), maxdim, pairs.data_ptr(), None, cap,
                                             offsets.data_ptr(), ctypes.byref(n),
                                             ctypes.c_void_p(stream.cuda_stream))
            cr._check(st)
            m = int(n.value)
            if world > 1:  # the job ends with every shard's barcodes gathered in input order
                from paper_2005_12692_b200.dist import gather_barcodes
                p_all, _ = gather_barcodes(pairs[:m], offsets)
                return int(p_all.shape[0])
            return m
        if f64:
            return len(cr.barcodes_f64(img, maxdim, capacity=cap).dim)
        return len(cr.barcodes(img, maxdim, out=(pairs, None)).pairs)

    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)  # 256 MiB > L2
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
    stage_tot = {}
    launches = 0
    for k in range(args.steps):
        flush.zero_()
        ev[k][0].record(stream)
        n_out = step()
        ev[k][1].record(stream)
        st = cr.last_stats()
        launches += st["launches"]
        for name, ms in st["stages"].items():
            stage_tot[name] = stage_tot.get(name, 0.0) + ms
    torch.cuda.synchronize()
    if dist.is_initialized():
        dist.barrier()
    torch.cuda.synchronize()
    clocks = sampler.stop() if sampler else None
    total_ms = sum(a.elapsed_time(b) for a, b in ev)
    if dist.is_initialized():
        t = torch.tensor([total_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    nvox_total = nvox_local * world if not batched else None
    if batched:
        full = int(np.prod(host_img.shape[1:])) * units_total
        nvox_total = full
    value = nvox_total / (ms_per_step / 1e3)

    # ---- end to end through the host entry point (pinned buffers, copies inside the region)
    e2e = None
    if batched:  # the shard's images from pinned host memory, bars + offsets back to the host
        pin_in = torch.from_numpy(np.ascontiguousarray(host_img)).pin_memory()
        dev_in = torch.empty_like(pin_in, device=dev)
        pin_pairs = torch.empty((cap, 3), dtype=torch.int32).pin_memory()
        pin_off = torch.empty((img.shape[0] + 1,), dtype=torch.int64).pin_memory()

        def e2e_step():  # (the gather of N > 1 happens inside step, on the devices)
            dev_in.copy_(pin_in, non_blocking=True)
            step(dev_in)
            pin_off.copy_(offsets, non_blocking=True)
            torch.cuda.current_stream(dev).synchronize()
            m = int(pin_off[-1])  # this shard's bars
            pin_pairs[:m].copy_(pairs[:m], non_blocking=True)
            torch.cuda.current_stream(dev).synchronize()
            return m
        for _ in range(max(1, args.warmup)):
            e2e_step()
        torch.cuda.synchronize()
        if dist.is_initialized():
            dist.barrier()
        e2e_ev = []
        m_out = 0
        for k in range(args.steps):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            m_out = e2e_step()
            b.record(stream)
            e2e_ev.append((a, b))
        torch.cuda.synchronize()
        e2e_ms = sum(a.elapsed_time(b) for a, b in e2e_ev)
        if dist.is_initialized():
            t = torch.tensor([e2e_ms], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_ms = float(t.item())
        e2e = {"value": (nvox_local * world) / (e2e_ms / args.steps / 1e3), "unit": "voxels/s",
               "h2d_bytes_per_step": nvox_local * 4,
               "d2h_bytes_per_step": m_out * 12 + (int(img.shape[0]) + 1) * 8,
               "ms_per_step": e2e_ms / args.steps}
    elif f64:  # public API with host buffers: pinned double in, float64 bars out
        pin_in = torch.from_numpy(np.ascontiguousarray(host_img)).pin_memory()
        dev_in = torch.empty_like(pin_in, device=dev)

        def e2e_step():
            dev_in.copy_(pin_in, non_blocking=True)
            bc = cr.barcodes_f64(dev_in, maxdim, capacity=cap)
            res = (bc.dim.cpu(), bc.birth.cpu(), bc.death.cpu())
            return len(res[0])
        for _ in range(max(1, args.warmup)):
            e2e_step()
        torch.cuda.synchronize()
        e2e_ev = []
        for k in range(args.steps):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            m_out = e2e_step()
            b.record(stream)
            e2e_ev.append((a, b))
        torch.cuda.synchronize()
        e2e_ms = sum(a.elapsed_time(b) for a, b in e2e_ev)
        if dist.is_initialized():
            t = torch.tensor([e2e_ms], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_ms = float(t.item())
        e2e = {"value": nvox_total / (e2e_ms / args.steps / 1e3), "unit": "voxels/s",
               "h2d_bytes_per_step": nvox_local * 8, "d2h_bytes_per_step": m_out * 20,
               "ms_per_step": e2e_ms / args.steps}
    elif not batched:
        pin_in = torch.from_numpy(np.ascontiguousarray(host_img)).pin_memory()
        pin_out = torch.empty((cap, 3), dtype=torch.int32).pin_memory()
        for _ in range(max(1, args.warmup)):
            cr.barcodes_host(pin_in, maxdim, out=(pin_out, None), stream=stream)
        torch.cuda.synchronize()
        if dist.is_initialized():
            dist.barrier()
        e2e_ev = []
        d2h = 0
        for k in range(args.steps):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            bc = cr.barcodes_host(pin_in, maxdim, out=(pin_out, None), stream=stream)
            b.record(stream)
            e2e_ev.append((a, b))
            d2h = len(bc.pairs) * 12
        torch.cuda.synchronize()
        e2e_ms = sum(a.elapsed_time(b) for a, b in e2e_ev)
        if dist.is_initialized():
            t = torch.tensor([e2e_ms], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_ms = float(t.item())
        e2e = {"value": nvox_total / (e2e_ms / args.steps / 1e3), "unit": "voxels/s",
               "h2d_bytes_per_step": nvox_local * 4, "d2h_bytes_per_step": d2h,
               "ms_per_step": e2e_ms / args.steps}

    if rank != 0:
        return None
    # ---- roofline of the dominant stage (per-stage CUDA events on the call's stream)
    hbm, peak_src = peaks()
    st = stats_warm
    K_basins = st["columns"][0]
    stage_avg = {k: v / args.steps for k, v in stage_tot.items()}
    dom = max(stage_avg, key=stage_avg.get) if stage_avg else None
    alg = algorithmic_bytes(args.config, dom, nvox_local, st, n_out,
                            None if batched else tuple(host_img.shape))
    # the filtration (K1) and apparent-pair (K2) kernels' achieved bandwidth (BASELINE north_star)
    k1k2 = None
    k12_names = [n for n in ("filtration", "births", "apparent") if n in stage_avg]
    if not batched and k12_names:
        k1k2 = {}
        if "filtration" in stage_avg:
            k1k2["fused"] = "K1 and K2 are one kernel (k_filtration): the entry covers both"
        for name in k12_names:
            b = algorithmic_bytes(args.config, name, nvox_local, st, n_out, tuple(host_img.shape))
            gbs = b / (stage_avg[name] / 1e3) / 1e9
            k1k2[name] = {"ms": round(stage_avg[name], 4), "alg_bytes": b,
                          "achieved_gbs": round(gbs, 1), "frac": round(gbs / hbm, 4)}
    roof = None
    if dom and alg:
        ach = alg / (stage_avg[dom] / 1e3) / 1e9
        roof = {"bound": "hbm", "kernel": dom, "achieved": round(ach, 1), "peak": hbm,
                "unit": "GB/s", "frac": round(ach / hbm, 4), "traffic": None,
                "alg_bytes_per_launch": alg, "avg_ms": round(stage_avg[dom], 5),
                "peak_source": peak_src}
        roof.update(ncu_traffic(dom))
        # The same kernel against the instruction-issue ceiling: warp instructions
        # per launch (ncu) / the live launch time, vs 148 SMs x 4 schedulers x 1 warp-instruction
        # per clock at the sampled SM clock.  The 1D and the fused K1+K2 kernels are issue-bound.
        wi = roof.pop("warp_instructions", None)
        if wi:
            mhz = (clocks or {}).get("sm_mhz") or 1965.0
            ipeak = 148 * 4 * mhz * 1e6 / 1e9  # G warp-instructions/s
            iach = wi / (stage_avg[dom] / 1e3) / 1e9
            roof["issue"] = {"achieved": round(iach, 1), "peak": round(ipeak, 1),
                             "unit": "G warp-inst/s", "frac": round(iach / ipeak, 4)}
    out = {
        "metric": METRIC, "value": value, "unit": "voxels/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64" if f64 else "f32",
        "data": "synthetic (seeded, workloads/generators.py)",
        "config": {"workload": f"{args.config}: {CONFIG_DESC[args.config]}",
                   "voxels_per_step": nvox_total, "maxdim": maxdim,
                   "parallelism": (f"dp{world} (image shards)" if batched else
                                   f"replicas x{world} (one image per rank)"),
                   "l2": "flushed before every timed step (256 MiB write, outside the events)",
                   "bars_per_step": n_out},
        "roofline": roof,
        "k1_k2": k1k2,
        "stages_ms": {k: round(v, 5) for k, v in stage_avg.items()},
        "clocks": clocks,
        "e2e": e2e,
        "gpu_launches": launches,
        "stats": {k: st[k] for k in ("cells", "apparent", "columns", "rounds", "pairs", "path")},
    }
    if world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(args.config, host_img, maxdim)
    return out


def algorithmic_bytes(cfg, stage, nvox, st, n_out, shape=None):
    """Bytes a stage must move once."""
    K = st["columns"][0]
    if stage is None:
        return None
    if stage == "1d_level1":
        return 4 * nvox + 8 * n_out               # read the series, stage (birth, death) per bar
    if stage == "1d_levels_gather":
        return 20 * n_out                         # read staged pairs, write 12-B output bars
    if stage.startswith("1d_count"):
        return 4 * nvox                           # read x
    if stage.startswith("1d_scatter"):
        return 4 * nvox + 24 * K                  # read x, write basin/barrier keys + cells
    if stage.startswith("1d_deaths"):
        return 24 * K                             # read basin+barrier keys, write death keys
    if stage.startswith("1d_emit"):
        return 28 * K + 12 * n_out                # read keys/death/cells, write bars
    if stage.startswith("1d_tree"):
        return 32 * K                             # read level 0, write levels >= 1 (~K)
    if stage in ("f64_rank", "f64_cast"):        # read the doubles, write the float32 surrogate
        return 12 * nvox + (8 * nvox if stage == "f64_rank" else 0)  # + table of distinct values
    if stage == "f64_map":
        return 12 * n_out + 24 * n_out            # read float32 bars, write float64 bars
    kcells = khalimsky_cells(shape) if shape else sum(st["cells"])
    if stage == "births":                         # read the image, write every Khalimsky cell
        return 4 * nvox + 4 * kcells
    if stage == "apparent":                       # read the births, write a tag per cell
        return 5 * kcells
    if stage == "filtration":                     # K1+K2 fused: read the image, write births+tags
        return 4 * nvox + 5 * kcells
    return None


NCU_KERNEL = {"1d_level1": "k1_level1", "1d_levels_gather": "k1_levels_coop",
              "filtration": "k_filtration"}


def ncu_traffic(stage):
    """DRAM bytes per launch of the stage's kernel from the committed ncu --set full capture
    (profiles/), or nothing if there is none for it."""
    import glob
    k = NCU_KERNEL.get(stage)
    if not k:
        return {}
    for p in sorted(glob.glob(os.path.join(ROOT, "profiles", "*", "*", "ncu_full_*_summary.json")),
                    reverse=True):
        try:
            with open(p) as f:
                d = json.load(f)["kernels"][k]
            out = {"traffic": round((d["dram_read_MB"] + d["dram_write_MB"]) * 1e6),
                   "traffic_source": os.path.relpath(p, ROOT)}
            if "warp_instructions" in d:
                out["warp_instructions"] = int(float(d["warp_instructions"]))
            return out
        except (KeyError, OSError, ValueError):
            continue
    return {}


def khalimsky_cells(shape):
    n = 1
    for v in shape:
        n *= 2 * int(v) - 1
    return n


def cpu_baseline(cfg, host_img, maxdim):
    """The oracle (single-threaded C++), as it stands, on a bounded sample of the workload."""
    import oracle
    oracle.build()
    if cfg in ("c2", "c2f64"):
        sample = host_img
        desc = f"full {cfg} series (2^24 samples), one run"
    elif cfg in BATCHED:
        sample = host_img[:64]
        desc = f"first 64 images of the {cfg} batch"
    elif cfg == "c5":
        sample = host_img[96:288, 96:288, 96:288]
        desc = "central 192^3 crop of C5"
    else:
        sample = host_img
        desc = f"full {cfg}, one run"
    t0 = time.perf_counter()
    if cfg in BATCHED:
        for im in sample:
            oracle.ph(im, maxdim)
    else:
        oracle.ph(sample, maxdim, dtype=sample.dtype)
    dt = time.perf_counter() - t0
    return {"value": float(np.prod(sample.shape)) / dt, "unit": "voxels/s", "cores": 1,
            "kind": "oracle", "sample": desc, "seconds": dt}


def run_reference(args, rank, world):
    """--impl reference: the CPU oracle timed on host cores; rank 0 only."""
    if rank != 0:
        return None
    import oracle
    oracle.build()
    host_img, maxdim, _ = make_input(args.config, 0, 1)
    if args.config in ("c2", "c2f64"):
        sample, desc = host_img[: 1 << 20], f"first 2^20 samples of {args.config} per step"
    elif args.config in BATCHED:
        sample, desc = host_img[:16], f"first 16 images of {args.config} per step"
    elif args.config == "c5":
        sample, desc = host_img[160:224, 160:224, 160:224], "central 64^3 crop of C5 per step"
    else:
        sample, desc = host_img, f"full {args.config} per step"

    def one():
        if args.config in BATCHED:
            for im in sample:
                oracle.ph(im, maxdim)
        else:
            oracle.ph(sample, maxdim, dtype=sample.dtype)

    for _ in range(args.warmup):
        one()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        one()
    dt = (time.perf_counter() - t0) / args.steps
    v = float(np.prod(sample.shape)) / dt
    return {"impl": "reference", "metric": METRIC, "value": v, "unit": "voxels/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64" if args.config in F64 else "f32", "data": "synthetic (seeded, workloads/generators.py)",
            "config": {"workload": f"{args.config}: {CONFIG_DESC[args.config]}", "maxdim": maxdim},
            "cpu_baseline": {"value": v, "unit": "voxels/s", "cores": 1, "kind": "oracle",
                             "sample": desc},
            "e2e": {"value": v, "unit": "voxels/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c2", choices=sorted(CONFIG_DESC))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
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
