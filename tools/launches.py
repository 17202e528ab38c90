"""Summarise an ncu --csv launch list (gpu__time_duration.sum [+ dram bytes])."""
import collections
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hdr, by = None, collections.OrderedDict()
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            e = by.setdefault(d["ID"], {"name": d["Kernel Name"], "grid": d["Grid Size"],
                                        "block": d["Block Size"]})
            e[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
    return list(by.values())


def main(path, show=60):
    ks = load(path)
    tot = sum(k["gpu__time_duration.sum"] for k in ks)
    agg = collections.defaultdict(lambda: [0.0, 0, 0.0])
    for k in ks:
        n = k["name"].split("(")[0].replace("hpsb::<unnamed>::", "")[:50]
        a = agg[n]
        a[0] += k["gpu__time_duration.sum"]
        a[1] += 1
        a[2] += k.get("dram__bytes_read.sum", 0) + k.get("dram__bytes_write.sum", 0)
    print(f"{len(ks)} launches, total {tot / 1e3:.1f} us")
    for n, (t, c, b) in sorted(agg.items(), key=lambda x: -x[1][0]):
        print(f"{t / 1e3:10.1f} us {100 * t / tot:5.1f}% x{c:4d} {b / 1e6:9.1f} MB "
              f"{b / max(t, 1):7.0f} GB/s  {n}")
    print("--- sequence")
    for i, k in enumerate(ks[:show]):
        t = k["gpu__time_duration.sum"]
        b = k.get("dram__bytes_read.sum", 0) + k.get("dram__bytes_write.sum", 0)
        print(f"{i:4d} {t / 1e3:8.1f} us {b / 1e6:8.1f} MB {b / max(t, 1):6.0f} GB/s "
              f"{k['grid']:>16} {k['name'].split('(')[0].replace('hpsb::<unnamed>::', '')[:40]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 60)
