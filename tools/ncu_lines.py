"""Stall samples and executed instructions per CUDA source line of one kernel
in an ncu report (needs -lineinfo and --import-source on):
    python tools/ncu_lines.py REPORT KERNEL_REGEX [TOP]"""
import collections
import csv
import subprocess
import sys


def main(rep, kern, top=30):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                          "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
    samples, instr, text = collections.Counter(), collections.Counter(), {}
    path, line, hdr = "?", None, None
    for r in csv.reader(out.splitlines()):
        if not r:
            continue
        if r[0] == "File Path":
            path = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < 8:
            continue
        if r[0]:
            line = (path, int(r[0]))
            text[line] = r[1].strip()[:90]
            continue
        try:
            samples[line] += float(r[4] or 0)
            instr[line] += float(r[7] or 0)
        except ValueError:
            pass
    tot = sum(samples.values()) or 1.0
    print(f"{kern}: {tot:.0f} samples, {sum(instr.values()):.0f} warp instructions")
    for ln, s in samples.most_common(top):
        print(f"{100 * s / tot:5.1f}% {instr[ln]:10.0f}  {ln[0]}:{ln[1]:<4d} {text.get(ln, '')}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 30)
