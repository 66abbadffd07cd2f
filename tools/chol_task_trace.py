"""Per-task timeline of Cholesky factorizations (ABD_CHOL_TRACE_TASKS=file): task-type
durations, concurrency profile and the waiting between a task becoming poppable and
starting.  Usage: python tools/chol_task_trace.py TRACE.bin [which factorization, default last]"""
import struct
import sys

import numpy as np


def load(path):
    data = open(path, "rb").read()
    out, off = [], 0
    while off < len(data):
        n, m, nt, grid, npart, nbo = struct.unpack_from("6i", data, off)
        off += 24
        rec = np.frombuffer(data, dtype=np.uint64, count=4 * nt, offset=off).reshape(nt, 4)
        off += 32 * nt
        fseq = None
        if npart < 0:  # k_chol_flow traces carry the forward items' codes
            fseq = np.frombuffer(data, dtype=np.int32, count=m + nbo, offset=off)
            off += 4 * (m + nbo)
        out.append((n, m, nt, grid, npart, nbo, rec, fseq))
    return out


def main():
    facs = load(sys.argv[1])
    k = int(sys.argv[2]) if len(sys.argv) > 2 else -1
    n, m, nt, grid, npart, nbo, rec, fseq = facs[k]
    rec = rec[rec[:, 3] > 0]
    item = (rec[:, 0] & 0xffffffff).astype(np.int64)
    info = (rec[:, 0] >> 32).astype(np.int64)
    tpop, ts, te = rec[:, 1].astype(np.int64), rec[:, 2].astype(np.int64), rec[:, 3].astype(np.int64)
    t0 = ts.min()
    if npart < 0:  # k_chol_flow: items [0, m + nbo) forward (diagonals and blocks), then backward
        npart = 0
        code = np.where(item < m + nbo, fseq[np.minimum(item, m + nbo - 1)], -1)
        kind = np.where(item < m + nbo, np.where(code < n, 0, 1), 2)
        names = ["diagonal", "block", "backward"]
        # the last diagonals in elimination order: completion times and what they waited for
        dsel = np.nonzero(kind == 0)[0]
        dsel = dsel[np.argsort(item[dsel])][-40:]
        print("  last 40 diagonals: end (us from start), ready->end (us), grab->ready (us)")
        print("   ", " ".join(f"{(te[i] - tpop.min()) / 1e3:.0f}/{(te[i] - ts[i]) / 1e3:.1f}/{(ts[i] - tpop[i]) / 1e3:.0f}"
                            for i in dsel))
        bsel = np.nonzero(kind == 1)[0]
        print(f"  blocks ready->end mean {(te[bsel] - ts[bsel]).mean() / 1e3:.2f} us; diagonals ready->end mean "
              f"{(te[kind == 0] - ts[kind == 0]).mean() / 1e3:.2f} us")
    else:
        kind = np.where(item < npart, 0, np.where(item < npart + nbo, 1, 2))
        names = ["partial/diag", "block", "backward"]
    print(f"{len(facs)} factorizations; this one: n={n} coupled={m} tasks={nt} (partials {npart}, blocks {nbo}) "
          f"grid={grid} CTAs, span {(te.max() - t0) / 1e3:.1f} us, busy {(te - ts).sum() / 1e3:.1f} warp-us")
    for kk in range(3):
        sel = kind == kk
        d = (te - ts)[sel]
        if sel.any():
            print(f"  {names[kk]:14s} n={sel.sum():6d} mean {d.mean() / 1e3:6.2f} us  p90 {np.percentile(d, 90) / 1e3:6.2f}"
                  f"  max {d.max() / 1e3:6.2f}  total {d.sum() / 1e3:8.1f} us  info mean {info[sel].mean():.1f} max {info[sel].max()}")
    # factor phase end = last non-backward end
    fend = te[kind < 2].max()
    print(f"  factor phase {(fend - t0) / 1e3:.1f} us, backward phase {(te.max() - fend) / 1e3:.1f} us")
    # concurrency profile in 10 us bins
    bins = np.arange(t0, te.max() + 10000, 10000)
    conc = np.zeros(len(bins) - 1)
    for a, b in zip(ts, te):
        i0, i1 = np.searchsorted(bins, a, "right") - 1, np.searchsorted(bins, b, "right") - 1
        for i in range(max(i0, 0), min(i1, len(conc) - 1) + 1):
            lo, hi = max(a, bins[i]), min(b, bins[i + 1])
            if hi > lo:
                conc[i] += (hi - lo) / 10000
    print("  mean running tasks per 10 us bin:", " ".join(f"{c:.1f}" for c in conc))
    # popped-but-waiting (polled a slot before it was filled) vs continuation
    wait = ts - tpop
    print(f"  pop->start wait: mean {wait.mean() / 1e3:.2f} us, p90 {np.percentile(wait, 90) / 1e3:.2f} us "
          f"(0 for continuations: {np.mean(wait == 0) * 100:.0f}% of tasks)")
    # tasks in the low-concurrency tail (last 30% of the factor phase)
    tail = (ts > t0 + 0.7 * (fend - t0)) & (kind < 2)
    for kk in range(2):
        sel = tail & (kind == kk)
        if sel.any():
            d = (te - ts)[sel]
            print(f"  tail {names[kk]:14s} n={sel.sum():5d} mean {d.mean() / 1e3:6.2f} us, info mean {info[sel].mean():.1f}")


if __name__ == "__main__":
    main()
