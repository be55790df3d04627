"""Summarise an ncu source page (cuda,sass) by source line / region.

usage: python tools/ncu_regions.py report.ncu-rep [file.cuh:first-last=name ...]
"""
import collections
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    regions = []
    for a in sys.argv[2:]:
        spec, name = a.split("=")
        f, rng = spec.split(":")
        lo, hi = map(int, rng.split("-"))
        regions.append((f, lo, hi, name))
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    fname = None
    tot_ie = tot_s = 0
    by_ie, by_s, lines = collections.Counter(), collections.Counter(), []
    reasons = collections.defaultdict(collections.Counter)
    hdr = None
    for r in csv.reader(io.StringIO(out)):
        if len(r) > 8 and r[0] == "Line No":
            hdr = r
            continue
        if len(r) == 2 and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if len(r) < 8 or r[0] in ("Line No", ""):
            continue
        try:
            s, ie = int(r[4]), int(r[7])
        except ValueError:
            continue
        tot_ie += ie
        tot_s += s
        reg = "other:" + fname
        for f, lo, hi, name in regions:
            if f == fname and lo <= int(r[0]) <= hi:
                reg = name
        by_ie[reg] += ie
        by_s[reg] += s
        if hdr:
            for i, h in enumerate(hdr):
                if h.startswith("stall_") and "Not Issued" not in h and i < len(r):
                    try:
                        reasons[reg][h[6:]] += int(r[i])
                    except ValueError:
                        pass
        lines.append((s, ie, f"{fname}:{r[0]}", r[1].strip()[:100]))
    print(f"total warp-instructions {tot_ie:.4g}, stall samples {tot_s}")
    for k in sorted(by_ie, key=lambda k: -by_s[k]):
        top = ", ".join(f"{n} {100 * v / max(1, by_s[k]):.0f}%" for n, v in reasons[k].most_common(4))
        print(f"  {k:28s} inst {100 * by_ie[k] / tot_ie:5.1f}%   samples {100 * by_s[k] / tot_s:5.1f}%   [{top}]")
    lines.sort(reverse=True)
    for s, ie, where, src in lines[:25]:
        print(f"  {100 * s / tot_s:5.1f}%  ie={ie:.3g}  {where}  {src}")


if __name__ == "__main__":
    main()
