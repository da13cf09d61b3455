"""Summarise a fused-qgZ tile timeline (ZPP_QGZ_TRACE=<prefix>): per kind
(P quantize / C intra fold / D inter fold) the tile count, mean busy time,
mean wait, and the kernel span; plus the per-SM tile-claim gaps."""
import sys
import numpy as np


def load(path):
    a = np.fromfile(path, dtype=np.uint64).reshape(-1, 4)
    return a


def main():
    for path in sys.argv[1:]:
        a = load(path)
        tile = (a[:, 0] & 0xFFFFFFFF).astype(np.int64)
        sm = ((a[:, 0] >> 32) & 0xFFFF).astype(np.int64)
        kind = (a[:, 0] >> 48).astype(np.int64)
        t0 = a[:, 1].min()
        start, wait, end = (a[:, 1] - t0) / 1e3, (a[:, 2] - t0) / 1e3, (a[:, 3] - t0) / 1e3
        print(path, "tiles", len(a), "span_us %.1f" % end.max())
        busy = end - wait
        w = wait - start
        for kd, name in ((0, "P"), (1, "C"), (2, "D")):
            m = kind == kd
            if m.any():
                print("  %s: %d tiles, busy mean %.2f us (p90 %.2f), wait mean %.2f us max %.1f, first start %.1f last end %.1f" %
                      (name, m.sum(), busy[m].mean(), np.percentile(busy[m], 90), w[m].mean(), w[m].max(),
                       start[m].min(), end[m].max()))
        order = np.argsort(start)
        # per-SM utilisation: sum(end-start)/span over SMs (two CTAs per SM)
        util = (end - start).sum() / (end.max() * len(np.unique(sm)) * 2)
        print("  CTA-slot utilisation %.2f" % util)
        # timeline in 10 buckets: tiles completed
        hist, edges = np.histogram(end, bins=10)
        print("  completions per 10% of span:", hist.tolist())
        np.save(path.replace(".bin", ".npy"), np.stack([tile, sm, kind, start, wait, end], 1))


if __name__ == "__main__":
    main()
