#!/usr/bin/env python3
"""Stall samples per CUDA source line of one kernel in an ncu report
(--page source, cuda+sass view): the top lines and their two main stall
reasons.  python tools/ncu_lines.py report.ncu-rep [top]"""
import collections
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    fname, cur, samp, stalls = None, None, None, []
    agg, srcs = collections.defaultdict(float), {}
    det = collections.defaultdict(collections.Counter)
    for r in csv.reader(io.StringIO(out)):
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Function Name":
            continue
        if r[0] == "Line No":
            idx = {}
            for k, h in enumerate(r):
                idx.setdefault(h, k)
            samp = idx["Warp Stall Sampling (All Samples)"]
            stalls = [(k, h) for k, h in enumerate(r) if h.startswith("stall_") and "Not Issued" not in h]
            continue
        if r[0].isdigit():
            cur = (fname, int(r[0]))
            srcs[cur] = r[1][:80]
            if r[2] == "-":
                continue
        try:
            s = float(r[samp] or 0)
        except (ValueError, TypeError):
            continue
        agg[cur] += s
        for k, h in stalls:
            try:
                det[cur][h] += float(r[k] or 0)
            except ValueError:
                pass
    tot = sum(agg.values()) or 1
    print(f"total samples {tot:.0f}")
    for key, s in sorted(agg.items(), key=lambda x: -x[1])[:top]:
        t2 = [(h[6:], round(v / tot * 100, 1)) for h, v in det[key].most_common(2)]
        print(f"{s / tot * 100:5.1f} {key[0]}:{key[1]} {srcs.get(key, '')} {t2}")


if __name__ == "__main__":
    main()
