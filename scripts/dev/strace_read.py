"""Summarise a LRS_STRACE file (development aid)."""
import sys

import numpy as np

raw = open(sys.argv[1], "rb").read()
o = 0
while o < len(raw):
    mode, nt = np.frombuffer(raw[o:o + 8], dtype=np.int32)
    o += 8
    a = np.frombuffer(raw[o:o + nt * 64], dtype=np.uint64).reshape(nt, 8).astype(np.int64)
    o += nt * 64
    t0 = a[:, 0].min()
    p = (a[:, 6] >> 32) * 64 + a[:, 7]  # chain = (partition, column group)
    t = a[:, 6] & 0xffffffff
    pub = a[:, 5] - t0
    print(f"mode {mode} tiles {nt} span {(a[:, 5].max() - t0) / 1e3:.1f} us")
    a = a[a[:, 5] > 0]
    p = (a[:, 6] >> 32) * 64 + a[:, 7]
    t = a[:, 6] & 0xffffffff
    steps, lat_flag, lat_dep, lat_diag, lat_pub, late = [], [], [], [], [], []
    for pp in np.unique(p):
        idx = np.flatnonzero(p == pp)
        idx = idx[np.argsort(t[idx] if mode == 0 else -t[idx])]
        for a1, b1 in zip(idx[:-1], idx[1:]):
            steps.append(a[b1, 5] - a[a1, 5])
            lat_flag.append(a[b1, 2] - a[a1, 5])       # publish(t-1) -> seen by t
            lat_dep.append(a[b1, 3] - a[b1, 2])        # x_{t-1} + last dep tile
            lat_diag.append(a[b1, 4] - a[b1, 3])       # diagonal product
            lat_pub.append(a[b1, 5] - a[b1, 4])        # write + fence + publish
            late.append(a[b1, 1] - a[a1, 5])           # >0: CTA arrived at last wait late
    for name, v in (("step", steps), ("flag", lat_flag), ("dep", lat_dep), ("diag", lat_diag),
                    ("publish", lat_pub), ("wait_begin-after-publish", late)):
        v = np.array(v) / 1e3
        print(f"  {name:26s} median {np.median(v):7.2f} us  p10 {np.percentile(v, 10):7.2f}  p90 {np.percentile(v, 90):7.2f}")
    frac_late = np.mean(np.array(late) > 0)
    print(f"  CTAs reaching last wait after the flag: {frac_late:.2f}")
