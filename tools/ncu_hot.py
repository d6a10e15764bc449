"""Summarise an ncu report's SASS page: top instructions by stall samples and by count.

usage: python tools/ncu_hot.py report.ncu-rep [kernel-regex] [top]
"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
    cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"]
    if len(sys.argv) > 2 and sys.argv[2]:
        cmd += ["-k", "regex:" + sys.argv[2]]
    out = subprocess.run(cmd, capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = next(r for r in rows if r and r[0] == "Address")
    body = [r for r in rows if len(r) == len(hdr) and r[0].startswith("0x")]
    ix = {h: i for i, h in enumerate(hdr)}
    samp = ix["Warp Stall Sampling (All Samples)"]
    ex = ix["Instructions Executed"]
    tot_s = sum(float(r[samp] or 0) for r in body)
    tot_e = sum(float(r[ex] or 0) for r in body)
    print(f"instructions {len(body)}  executed {tot_e:.3e}  samples {tot_s:.0f}")
    # 16-instruction windows by samples
    win = []
    for i in range(0, len(body), 16):
        s = sum(float(r[samp] or 0) for r in body[i:i + 16])
        e = sum(float(r[ex] or 0) for r in body[i:i + 16])
        win.append((s, e, i))
    print("hot windows (index, samples%, executed%):")
    for s, e, i in sorted(win, reverse=True)[:12]:
        print(f"  [{i:5d}] {100 * s / tot_s:5.1f}%  {100 * e / tot_e:5.1f}%  {body[i][1].strip()[:60]}")
    print("top instructions by samples:")
    for r in sorted(body, key=lambda r: -float(r[samp] or 0))[:top]:
        print(f"  {body.index(r):5d} {100 * float(r[samp] or 0) / tot_s:5.1f}%  ex={float(r[ex] or 0):.2e}  {r[1].strip()[:70]}")


if __name__ == "__main__":
    main()


def windows_by_executed(rep, width=32, top=20):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = next(r for r in rows if r and r[0] == "Address")
    body = [r for r in rows if len(r) == len(hdr) and r[0].startswith("0x")]
    ex = hdr.index("Instructions Executed")
    tot = sum(float(r[ex] or 0) for r in body)
    w = [(sum(float(r[ex] or 0) for r in body[i:i + width]), i) for i in range(0, len(body), width)]
    for e, i in sorted(w, reverse=True)[:top]:
        print(f"  [{i:5d}] {100 * e / tot:5.1f}%  {body[i][1].strip()[:60]}")
    return body
