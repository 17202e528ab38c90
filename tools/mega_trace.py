"""Summarise an HPSB_MEGA_TRACE file: per segment first start / last end /
mean task time / mean wait, relative to the launch's first task start (us)."""
import sys
from collections import defaultdict


def main(path):
    lines = open(path).read().splitlines()
    i = 0
    while i < len(lines):
        if not lines[i].startswith("launch"):
            i += 1
            continue
        print(lines[i])
        i += 1
        segs = []
        while lines[i].startswith("seg"):
            f = dict(kv.split("=") for kv in lines[i].split()[2:])
            a, b = map(int, f["tasks"].split(":"))
            segs.append((lines[i], a, b))
            i += 1
        rows = []
        while i < len(lines) and lines[i] and lines[i][0].isdigit():
            t, s, w, e = map(int, lines[i].split())
            rows.append((t, s, w, e))
            i += 1
        t0 = min(r[1] for r in rows if r[1])
        for desc, a, b in segs:
            rs = [r for r in rows if a <= r[0] < a + b]
            st = min(r[1] for r in rs) - t0
            en = max(r[3] for r in rs) - t0
            dur = sum(r[3] - r[1] for r in rs) / len(rs)
            wt = sum(r[2] - r[1] for r in rs) / len(rs)
            print(f"{desc:70s} start {st / 1e3:7.1f} end {en / 1e3:7.1f} task {dur / 1e3:6.2f} wait {wt / 1e3:6.2f} us")


if __name__ == "__main__":
    main(sys.argv[1])
