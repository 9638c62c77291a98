"""Time cr_barcodes on BASELINE configs and check the bars against the oracle digests.

Usage: python tools/time_configs.py c4 c5 c5b [--reps 3] [--debug]
Prints one JSON line per config: ms per call (min/median over reps, CUDA events around the call),
per-stage device times, cr_stats counters, and whether the bars' SHA-256 equals the oracle's
(tests/golden/fullsize_oracle.json).  Measurement helper only; the tests are the parity gate.
"""
import hashlib
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
if "--pkgroot" in sys.argv:  # a copy of the package with a variant libcr.so (measurement only)
    sys.path.insert(0, sys.argv[sys.argv.index("--pkgroot") + 1])
import paper_2005_12692_b200 as cr  # noqa: E402
from workloads import generators as gen  # noqa: E402


def digest(d, b, e, c):
    h = hashlib.sha256()
    for a, t in ((d, np.int32), (b, np.float32), (e, np.float32), (c, np.uint32)):
        h.update(np.ascontiguousarray(a).view(t).tobytes())
    return h.hexdigest()


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--") and not a.startswith("/")]
    reps = 3
    if "--reps" in sys.argv:
        reps = int(sys.argv[sys.argv.index("--reps") + 1])
        args = [a for a in args if a != str(reps)]
    gold = json.load(open(os.path.join(ROOT, "tests", "golden", "fullsize_oracle.json")))
    if "--debug" in sys.argv:
        cr.set_option("debug", 1)
    if "--debug2" in sys.argv:
        cr.set_option("debug", 2)
    if "--debug3" in sys.argv:
        cr.set_option("debug", 3)
    cr.set_profiling(True)
    for name in args:
        img, md = gen.config(name)
        t = torch.from_numpy(img).cuda()
        batched = name in ("c3", "c5b")
        times = []
        for r in range(reps + 1):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            if batched:
                bc, off = cr.barcodes_batched(t, md, cells=True)
            else:
                bc = cr.barcodes(t, md, cells=True)
            e1.record()
            torch.cuda.synchronize()
            if r:
                times.append(e0.elapsed_time(e1))
        st = cr.last_stats()
        d, b, e, c = bc.numpy()
        if batched and name == "c5b":
            off = off.cpu().numpy()
            ok = all(digest(d[off[i]:off[i + 1]], b[off[i]:off[i + 1]], e[off[i]:off[i + 1]],
                            c[off[i]:off[i + 1]]) == v["bars"]
                     for i, v in enumerate(gold["c5b"]["volumes"]))
        elif batched:
            ok = None
        else:
            ok = digest(d, b, e, c) == gold[name]["bars"]
        rec = {"config": name, "ms_min": round(min(times), 3),
               "ms_med": round(float(np.median(times)), 3), "times": [round(x, 2) for x in times],
               "bars": int(len(d)), "oracle_digest_ok": ok, "stats": st}
        print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
