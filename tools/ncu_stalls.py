"""Summarise an ncu source-page CSV (``--page source --csv --print-source sass``):
top instructions by warp-stall samples with their dominant stall reasons.
Addresses are printed relative to the kernel's first instruction.

    python tools/ncu_stalls.py src.csv [top] [off_lo off_hi]
"""
import csv
import sys


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    lo, hi = (int(sys.argv[3], 16), int(sys.argv[4], 16)) if len(sys.argv) > 4 else (0, 1 << 62)
    hdr = rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    base = int(rows[2][0], 16)
    body = [r for r in rows[2:] if len(r) == len(hdr) and lo <= int(r[0], 16) - base < hi]
    col = ix["Warp Stall Sampling (All Samples)"]
    tot = sum(int(r[col] or 0) for r in body)
    agg = {k: sum(int(r[ix[k]] or 0) for r in body) for k in reasons}
    print("total samples", tot)
    print("by reason", sorted(((v, k) for k, v in agg.items() if v), reverse=True)[:10])
    order = sorted(body, key=lambda r: -int(r[col] or 0))
    for r in order[:top]:
        s = int(r[col] or 0)
        why = sorted(((int(r[ix[k]] or 0), k[6:]) for k in reasons if int(r[ix[k]] or 0)), reverse=True)[:3]
        print(f"{int(r[0], 16) - base:6x} {s:6d} {100.0 * s / max(tot, 1):5.1f}%  {r[1].strip()[:56]:56s} {why}")


if __name__ == "__main__":
    main()
