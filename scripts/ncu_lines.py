"""Warp-stall samples of one kernel per source line.

ncu's SASS source page (``ncu -i X.ncu-rep --page source --csv --print-source sass``)
carries per-instruction stall samples but no line info; ``nvdisasm -g -c`` of the
kernel's cubin carries the line of every instruction offset.  This joins them.

usage: python scripts/ncu_lines.py sass_page.csv kernel.dis [top]
"""
import collections
import csv
import re
import sys


def main():
    src, dis = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
    rows = list(csv.reader(open(src)))
    hdr_i = next(i for i, r in enumerate(rows) if "Warp Stall Sampling (All Samples)" in r)
    h, body = rows[hdr_i], rows[hdr_i + 1:]
    i_all = h.index("Warp Stall Sampling (All Samples)")
    reasons = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
    ri = [h.index(c) for c in reasons]
    base = int(body[0][0], 16)
    line_of, cur = {}, None
    for ln in open(dis):
        m = re.search(r'File "([^"]+)", line (\d+)', ln)
        if m:
            cur = f"{m.group(1).rsplit('/', 1)[-1]}:{m.group(2)}"
            continue
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
        if m:
            line_of[int(m.group(1), 16)] = (cur, m.group(2).strip())
    agg = collections.defaultdict(lambda: collections.Counter())
    ops = collections.defaultdict(collections.Counter)
    total = 0.0
    for r in body:
        if not r or not r[0].startswith("0x"):
            continue
        s = float(r[i_all] or 0)
        total += s
        where, op = line_of.get(int(r[0], 16) - base, ("?", r[1]))
        agg[where]["all"] += s
        for c, i in zip(reasons, ri):
            agg[where][c] += float(r[i] or 0)
        ops[where][op.split()[0] if op else "?"] += s
    print(f"total samples {total:.0f}")
    for where, c in sorted(agg.items(), key=lambda kv: -kv[1]["all"])[:top]:
        rs = sorted(((k, v) for k, v in c.items() if k != "all" and v > 0), key=lambda kv: -kv[1])[:3]
        top_ops = ", ".join(f"{o}:{v:.0f}" for o, v in ops[where].most_common(2))
        print(f"{c['all'] / total * 100:5.1f}%  {where:28s} " + " ".join(f"{k[6:]}={v:.0f}" for k, v in rs) +
              f"   [{top_ops}]")


if __name__ == "__main__":
    main()
