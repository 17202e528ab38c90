"""Per-kernel DRAM traffic per launch from an ncu --csv launch list with
dram__bytes_read.sum / dram__bytes_write.sum (the bench command's timed
region), merged into profiles/traffic_kernels.json under the config name:
{config: {kernel: bytes per launch}} -- bench.py's roofline.traffic."""
import collections
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from launches import load  # noqa: E402


def norm(name):
    n = name.split("(")[0]
    for junk in ("void ", "hpsb::<unnamed>::", "hpsb::(anonymous namespace)::", "hpsb::"):
        n = n.replace(junk, "")
    return n.strip()


def main(csv_path, config, out=os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "profiles",
                                            "traffic_kernels.json")):
    agg = collections.defaultdict(lambda: [0.0, 0, 0.0])
    for k in load(csv_path):
        a = agg[norm(k["name"])]
        a[0] += k.get("dram__bytes_read.sum", 0) + k.get("dram__bytes_write.sum", 0)
        a[1] += 1
        a[2] += k["gpu__time_duration.sum"]
    try:
        with open(out) as fh:
            d = json.load(fh)
    except (OSError, ValueError):
        d = {}
    d[config] = {n: b / c for n, (b, c, _) in agg.items() if c}
    d[config + "/us_per_launch_ncu"] = {n: t / c / 1e3 for n, (_, c, t) in agg.items() if c}
    with open(out, "w") as fh:
        json.dump(d, fh, indent=1, sort_keys=True)
    for n, (b, c, t) in sorted(agg.items(), key=lambda kv: -kv[1][2]):
        print(f"{n:40s} x{c:4d} {b / c / 1e6:9.2f} MB/launch {t / c / 1e3:8.1f} us/launch")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
