"""Basic-block summary of an ncu SASS source export (csv or csv.gz): executed instructions, stall
samples and the opcode mix per run of instructions with the same execution count.

usage: python tools/sass_blocks.py export.csv[.gz] [min_share_pct]
"""
import collections
import csv
import gzip
import io
import re
import sys


def main():
    path = sys.argv[1]
    min_share = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
    text = gzip.open(path, "rt").read() if path.endswith(".gz") else open(path).read()
    rows = list(csv.reader(io.StringIO(text)))
    hdr = next(r for r in rows if r and r[0] == "Address")
    body = [r for r in rows if len(r) == len(hdr) and r[0].startswith("0x")]
    ix = {h: i for i, h in enumerate(hdr)}
    ex, sm = ix["Instructions Executed"], ix["Warp Stall Sampling (All Samples)"]
    stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    tot_e = sum(float(r[ex] or 0) for r in body)
    tot_s = sum(float(r[sm] or 0) for r in body)
    print(f"instructions {len(body)}  executed {tot_e:.4e}  samples {tot_s:.0f}")
    ops = collections.Counter()
    for r in body:
        m = re.match(r"\s*(@!?U?P\d+\s+)?([A-Z0-9_]+)", r[1])
        ops[m.group(2) if m else "?"] += float(r[ex] or 0)
    print("opcode mix (executed %):", ", ".join(f"{k} {100 * v / tot_e:.1f}" for k, v in ops.most_common(22)))
    st = collections.Counter()
    for r in body:
        for h in stall_cols:
            st[h] += float(r[ix[h]] or 0)
    print("stalls (%):", ", ".join(f"{k[6:]} {100 * v / tot_s:.1f}" for k, v in st.most_common(9)))
    # blocks: consecutive instructions whose execution counts are within 2 %
    blocks = []
    start = 0
    for i in range(1, len(body) + 1):
        if i == len(body) or abs(float(body[i][ex] or 0) - float(body[start][ex] or 0)) > 0.02 * max(
                1.0, float(body[start][ex] or 0)):
            blocks.append((start, i))
            start = i
    print("blocks (first, count, exec/instr, executed %, samples %, mix):")
    for a, b in blocks:
        e = sum(float(r[ex] or 0) for r in body[a:b])
        s = sum(float(r[sm] or 0) for r in body[a:b])
        if 100 * e / tot_e < min_share and 100 * s / tot_s < min_share:
            continue
        mix = collections.Counter()
        for r in body[a:b]:
            m = re.match(r"\s*(@!?U?P\d+\s+)?([A-Z0-9_]+)", r[1])
            mix[m.group(2) if m else "?"] += 1
        top = " ".join(f"{k}{v}" for k, v in mix.most_common(7))
        bs = collections.Counter()
        for r in body[a:b]:
            for h in stall_cols:
                bs[h[6:]] += float(r[ix[h]] or 0)
        tops = " ".join(f"{k}:{100 * v / max(s, 1):.0f}" for k, v in bs.most_common(3))
        print(f"  [{a:5d}] n={b - a:4d} x{float(body[a][ex] or 0):9.0f}  {100 * e / tot_e:5.1f}%  {100 * s / tot_s:5.1f}%  {top} | {tops}")


if __name__ == "__main__":
    main()
