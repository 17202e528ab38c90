"""Summarise an HPSB_MEGA_TRACE file: per segment first start / last end and
the mean task phases (us): wait for inputs, stage (gather), stream (columns),
finish (group sums, split partials, epilogue; emitting tasks only), relative
to the launch's first task start."""
import sys


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
            rows.append(list(map(int, lines[i].split())))
            i += 1
        t0 = min(r[1] for r in rows if r[1])
        for desc, a, b in segs:
            rs = [r for r in rows if a <= r[0] < a + b]
            st = min(r[1] for r in rs) - t0
            en = max(r[-1] for r in rs) - t0
            n = len(rs)
            mean = lambda j, k, sel=rs: sum(r[k] - r[j] for r in sel) / max(1, len(sel)) / 1e3
            em = [r for r in rs if len(r) > 6 and r[5]]
            if len(rs[0]) > 6:
                print(f"{desc[:60]:60s} {st / 1e3:6.1f}-{en / 1e3:6.1f} wait {mean(1, 2):5.2f} stage {mean(2, 3):5.2f}"
                      f" stream {mean(3, 4):5.2f} finish {mean(4, 5, em):5.2f} (emit {len(em)}/{n}) us")
            else:
                print(f"{desc[:60]:60s} {st / 1e3:6.1f}-{en / 1e3:6.1f} task {mean(1, 3):6.2f} wait {mean(1, 2):6.2f} us")


if __name__ == "__main__":
    main(sys.argv[1])
