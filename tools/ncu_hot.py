"""Summarise an `ncu --page source --csv` export (SASS view): stall totals and
the hottest instructions.  usage: python tools/ncu_hot.py <x.source.csv> [top]"""
import csv
import sys


def main():
    path = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    recs = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]
    stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    tot = {h: sum(float(r[h] or 0) for r in recs) for h in stall_cols}
    S = sum(tot.values()) or 1
    print("stall totals:", ", ".join(f"{k[6:]}={v / S:.2f}" for k, v in sorted(tot.items(), key=lambda x: -x[1]) if v / S > 0.01))
    key = "Warp Stall Sampling (All Samples)"
    recs.sort(key=lambda r: -float(r[key] or 0))
    for r in recs[:top]:
        st = sorted(((h[6:], float(r[h] or 0)) for h in stall_cols), key=lambda x: -x[1])[:3]
        print(f"{r[key]:>6} {r['Address'][-5:]} {r['Source'].strip()[:60]:60s} " + " ".join(f"{a}={b:.0f}" for a, b in st if b))


if __name__ == "__main__":
    main()
