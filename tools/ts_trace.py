"""Analyse a K1-TC-sym trace (a diagnostic patch, not kept in the product kernel:
%globaltimer stamps per chunk of warp 0 of each epilogue warpgroup): per warpgroup, the
time its warp 0 waits for each chunk's distance GEMM (S1FULL), for the chunk's
stage (SFULL) and works on the chunk, split by first-chunk-of-row vs others."""
import os, sys
import numpy as np
path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/ts_trace.bin"
h = np.fromfile(path, dtype=np.uint64).reshape(8, 4096)
for w in range(8):
    n = int(h[w, 0])
    if n == 0:
        continue
    t = h[w, 8:8 + 5 * n].reshape(n, 5)
    row = t[:, 4].astype(int)
    t3 = t[:, 3].astype(np.int64)
    t0, t1, t2 = t[:, 0].astype(np.int64), t[:, 1].astype(np.int64), t[:, 2].astype(np.int64)
    span = t3[-1] - t0[0]
    wg = t1 - t0
    ws = t2 - t1
    work = t3 - t2
    gap = np.r_[0, t0[1:] - t3[:-1]]
    first = np.r_[True, row[1:] != row[:-1]]
    print(f"wg {w}: {n} chunks, {row.max() + 1} rows, span {span / 1e3:.1f} us; "
          f"GEMM wait {wg.sum() / span:.1%} (row starts {wg[first].sum() / span:.1%}), "
          f"stage wait {ws.sum() / span:.1%}, work {work.sum() / span:.1%}, between chunks {gap.sum() / span:.1%} "
          f"(row ends {gap[first].sum() / span:.1%}); median work {np.median(work) / 1e3:.2f} us, "
          f"median GEMM wait {np.median(wg) / 1e3:.2f} us")
