"""Summarise the per-step timeline of a speculative greedy level
(IMB_SPEC_LOG output of greedy_spec.cu): median kernel durations and step
period per k range."""
import sys

import numpy as np


def main(path):
    for blk in open(path).read().split("# level")[1:]:
        lines = blk.strip().split("\n")
        d = np.array([[float(x) for x in l.split()] for l in lines[1:]])
        if len(d) < 500:
            continue
        print(lines[0])
        k = d[:, 0]
        insB, insE, solB, solE, fswE, swB, swE, chB, chE = d[:, 7:].T
        miss = (d[:, 4] != d[:, 6]) & (d[:, 4] >= 0)
        for lo, hi in [(100, 200), (1000, 1100), (2500, 2600), (4000, 4100), (4900, 5000)]:
            m = (k >= lo) & (k < hi)
            if not m.any():
                continue

            def med(x):
                x = x[m]
                x = x[x >= 0]
                return np.median(x) if len(x) else -1

            per = np.diff(swE, prepend=np.nan)
            print(f" k~{lo}: predict(ins+solve) {med(solE - insB):.0f} us (ins {med(insE - insB):.0f})"
                  f" fsweep {med(fswE - solE):.0f} sweep {med(swE - swB):.0f} chain {med(chE - chB):.0f}"
                  f" | sweep period {med(per):.0f} us | chainE->sweepB {med(swB - chE):.0f}"
                  f" | misses {int(miss[m].sum())}")


if __name__ == "__main__":
    main(sys.argv[1])
