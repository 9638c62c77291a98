"""Write tests/golden/fullsize_oracle.json: SHA-256 digests of the ORACLE's full-size results.

Calls only ``oracle/`` (and the seeded generators in ``workloads/``): no value here comes from
the CUDA path.  The oracle is the explicit boundary-matrix Z/2 reduction of PAPER.md:97-108,
130-142 (see oracle/cr_oracle.cpp); C5 takes ~3 min and ~20 GB on one core, so it is run once,
here, and the GPU tests (tests/test_gpu_fullsize.py) compare hashes of their own outputs with
these digests (the paper's own bar: outputs that coincide with an independent program,
PAPER.md:290).

Digested arrays (little-endian raw bytes, in the oracle's output order (dim, birth cell)):
  dim int32, birth float32, death float32, cell uint32 -- one digest over their concatenation
  (``bars``) -- and the partner array uint32 over kidx (``partner``).

Usage: python tools/oracle_digest.py [c5] [c5b] [c2] [c3] [c1] [c4]   (default: all)
"""
from __future__ import annotations

import hashlib
import json
import os
import resource
import sys
import time
from multiprocessing import Pool

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from workloads import generators as gen  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "fullsize_oracle.json")


def bars_digest(dim, birth, death, cell) -> str:
    h = hashlib.sha256()
    for a, t in ((dim, np.int32), (birth, np.float32), (death, np.float32), (cell, np.uint32)):
        h.update(np.ascontiguousarray(a).view(t).tobytes())
    return h.hexdigest()


def arr_digest(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _record(r, with_partner: bool) -> dict:
    rec = {"n_bars": int(len(r.dim)), "bars": bars_digest(r.dim, r.birth, r.death, r.cell),
           "per_dim": [[int(x) for x in row] for row in r.stats]}
    if with_partner:
        rec["partner"] = arr_digest(r.partner)
    return rec


def _one(args):
    img, md, partner = args
    return _record(oracle.ph(img, md, partner=partner), partner)


def run(name: str) -> dict:
    t0 = time.time()
    if name in ("c1", "c2", "c4", "c5"):
        img, md = gen.config(name)
        t1 = time.time()
        r = oracle.ph(img, md, partner=True)
        t2 = time.time()
        rec = _record(r, True)
        rec.update(gen_s=round(t1 - t0, 1), oracle_s=round(t2 - t1, 1))
    elif name == "c5b":
        vols, md = gen.config("c5b")
        t1 = time.time()
        with Pool(min(8, os.cpu_count() or 1)) as pool:
            recs = pool.map(_one, [(v, md, True) for v in vols], chunksize=1)
        rec = {"volumes": recs, "gen_s": round(t1 - t0, 1), "oracle_s": round(time.time() - t1, 1)}
    elif name == "c3":
        imgs, md = gen.config("c3")
        t1 = time.time()
        with Pool(min(8, os.cpu_count() or 1)) as pool:
            recs = pool.map(_one, [(im, md, i < 1024) for i, im in enumerate(imgs)],
                            chunksize=256)
        h = hashlib.sha256()
        for x in recs:
            h.update(x["bars"].encode())
        rec = {"images": len(recs), "bars_of_digests": h.hexdigest(),
               "partner_first1024": [x["partner"] for x in recs[:1024]],
               "n_bars": [x["n_bars"] for x in recs],
               "gen_s": round(t1 - t0, 1), "oracle_s": round(time.time() - t1, 1)}
    else:
        raise SystemExit(f"unknown config {name}")
    rec["maxrss_gb"] = round(resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 2 ** 20, 2)
    return rec


def main(names):
    data = {}
    if os.path.exists(OUT):
        with open(OUT) as f:
            data = json.load(f)
    data.setdefault("_about", "SHA-256 of the oracle's (oracle/) full-size outputs, written by "
                    "tools/oracle_digest.py; bars = sha256(dim i32 || birth f32 || death f32 || "
                    "cell u32) in (dim, birth cell) order; partner = sha256(partner u32)")
    for n in names:
        rec = run(n)
        data[n] = rec
        print(n, {k: v for k, v in rec.items() if k not in ("volumes", "partner_first1024",
                                                            "n_bars")}, flush=True)
        with open(OUT + ".tmp", "w") as f:
            json.dump(data, f, indent=1)
        os.replace(OUT + ".tmp", OUT)


if __name__ == "__main__":
    main(sys.argv[1:] or ["c1", "c2", "c4", "c3", "c5b", "c5"])
