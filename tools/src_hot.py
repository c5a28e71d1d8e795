"""Summarise an ncu `--page source --csv --print-source cuda,sass` export: per CUDA source line,
warp-stall samples and warp instructions executed (top N by samples).
  python tools/src_hot.py src.csv [N]"""
import csv
import sys


def main():
    path = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    f = None
    agg = {}
    hdr = None
    for r in csv.reader(open(path)):
        if not r:
            continue
        if r[0] == "File Path":
            f = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or r[0] == "" or r[0] == "Function Name":
            continue
        try:
            s = int(r[4]); ie = int(r[7])
        except (ValueError, IndexError):
            continue
        stalls = {hdr[i]: int(r[i]) for i in range(30, min(len(hdr), 47)) if r[i].isdigit() and int(r[i]) > 0}
        key = (f, int(r[0]))
        a = agg.setdefault(key, [0, 0, r[1][:90], {}])
        a[0] += s; a[1] += ie
        for k, v in stalls.items():
            a[3][k] = a[3].get(k, 0) + v
    tot_s = sum(a[0] for a in agg.values()); tot_i = sum(a[1] for a in agg.values())
    print(f"total samples {tot_s}, warp instructions {tot_i}")
    for (fn, ln), (s, ie, src, st) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
        tops = ",".join(f"{k.replace('stall_', '')}:{v * 100 // max(s, 1)}" for k, v in sorted(st.items(), key=lambda x: -x[1])[:3])
        print(f"{100 * s / tot_s:5.1f}% smp {100 * ie / tot_i:5.1f}% ins  {fn}:{ln:<5} {src.strip()[:70]:70s} {tops}")


if __name__ == "__main__":
    main()
