"""Claimant windows of the select kernel's blocks: for each
block of 256 consecutive parent slots, the offspring rows that can claim one
of its slots (rows c with B[c] meeting the block), merged into ranges with a
gap tolerance.  Prints the staged-row and range-count distribution.

    python tools/select_windows.py [PROBLEM N]
"""
import sys

import numpy as np

import paper_2509_19821_b200 as g


def windows(B, bs=256, gap=16):
    n, t = B.shape
    c = np.repeat(np.arange(n, dtype=np.int64), t)
    blk = B.reshape(-1).astype(np.int64) // bs
    key = np.unique(blk * n + c)
    blk, c = key // n, key % n
    # new range where the block changes or the gap to the previous row exceeds `gap`
    brk = np.ones(len(c), bool)
    brk[1:] = (blk[1:] != blk[:-1]) | (c[1:] - c[:-1] > gap)
    starts = np.flatnonzero(brk)
    ends = np.append(starts[1:], len(c)) - 1
    rb = blk[starts]
    rlen = c[ends] - c[starts] + 1
    nblk = (n + bs - 1) // bs
    rows = np.bincount(rb, weights=rlen, minlength=nblk)
    cnt = np.bincount(rb, minlength=nblk)
    return rows, cnt


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "LIRCMOP13"
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 1_000_000
    eng = g.Engine(g.make_problem(name), g.RunConfig(n=n, k_max=1, seed=1))
    topo = eng.neighborhoods()
    for q, B in ((1, topo.b1), (2, topo.b2)):
        for gap in (0, 8, 32):
            rows, cnt = windows(np.asarray(B), gap=gap)
            print(f"{name} N={n} pop{q} t={B.shape[1]} gap={gap}: staged rows per block mean {rows.mean():.0f} "
                  f"p99 {np.percentile(rows, 99):.0f} max {rows.max():.0f}; ranges mean {cnt.mean():.1f} "
                  f"p99 {np.percentile(cnt, 99):.0f} max {cnt.max()}", flush=True)


if __name__ == "__main__":
    main()
