"""Summarise VPG_TRACE tile-pipeline records (kernels.cu trace_begin/end,
tile_body.cuh trc[]): per launch, when CTAs start, when their first tile's
data is ready, how long W phases take, how long CTAs wait for data, and
when they finish -- all relative to the earliest CTA start (ns, globaltimer).

usage: VPG_TRACE=/tmp/t.bin python tools/quick_cfgs.py cfg3; python tools/trace_view.py /tmp/t.bin [launch]
"""
import sys

import numpy as np


def launches(path):
    raw = np.fromfile(path, dtype=np.uint64)
    i = 0
    while i + 3 <= raw.size:
        grid, ntiles, words = (int(x) for x in raw[i:i + 3])
        i += 3
        rec = raw[i:i + grid * words].reshape(grid, words)
        i += grid * words
        yield grid, ntiles, rec


def pct(a, qs=(0, 10, 50, 90, 100)):
    a = np.asarray(a, dtype=np.float64)
    if a.size == 0:
        return "-"
    return " ".join(f"p{q}={np.percentile(a, q) / 1e3:.2f}" for q in qs)


def summarise(grid, ntiles, rec):
    kw = rec.shape[1]
    start = rec[:, 0].astype(np.int64)
    ok = start > 0
    rec, start = rec[ok], start[ok]
    t0 = start.min()
    end = rec[:, 2].astype(np.int64)
    ntile = rec[:, kw - 1].astype(np.int64)
    pro = rec[:, 1].astype(np.int64)
    ready, done, waits = [], [], []
    first_ready = []
    for c in range(rec.shape[0]):
        prev = None
        for k in range(min(int(ntile[c]), 19)):
            r, w = int(rec[c, 4 + 3 * k + 1]), int(rec[c, 4 + 3 * k + 2])
            if r == 0 or w == 0:
                break
            ready.append(r - t0)
            done.append(w - r)
            if k == 0:
                first_ready.append(r - start[c])
            if prev is not None:
                waits.append(r - prev)
            prev = w
    sms = np.unique(rec[:, 3]).size
    print(f"grid {grid} ({rec.shape[0]} traced CTAs on {sms} SMs), tiles {ntiles}, tiles/CTA {pct(ntile * 1000)} (x1000)")
    print(f"  kernel span (first CTA start -> last CTA end): {(end.max() - t0) / 1e3:.2f} us")
    print(f"  CTA start after first (us):      {pct(start - t0)}")
    print(f"  first load issue after start:    {pct(rec[:, kw - 2].astype(np.int64) - start)}")
    print(f"  prologue issued after start:     {pct(pro - start)}")
    print(f"  first tile ready after start:    {pct(first_ready)}")
    print(f"  W phase per tile:                {pct(done)}")
    print(f"  wait for next tile after W:      {pct(waits)}")
    print(f"  CTA end (us from first start):   {pct(end - t0)}")
    print(f"  CTA busy (end - start):          {pct(end - start)}")


if __name__ == "__main__":
    want = int(sys.argv[2]) if len(sys.argv) > 2 else -1
    ls = list(launches(sys.argv[1]))
    print(f"{len(ls)} launches traced")
    for i, (g, n, r) in enumerate(ls):
        if want < 0 and i != len(ls) - 1:
            continue
        if want >= 0 and i != want:
            continue
        summarise(g, n, r)
