"""Split the SASS of one kernel (ncu --page source --print-source sass --csv) at
its BAR.SYNC / EXIT instructions and report warp-stall samples, instructions
and shared-memory wavefronts per segment (phase attribution for profiles/)."""
import csv
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    body = [r for r in rows[2:] if len(r) == len(hdr)]

    def f(r, k):
        v = r[ix[k]].replace(",", "")
        try:
            return float(v)
        except ValueError:
            return 0.0

    cuts = [0]
    for i, r in enumerate(body):
        s = r[ix["Source"]]
        if "BAR.SYNC" in s or "BAR.RED" in s or s.strip().startswith("EXIT"):
            cuts.append(i + 1)
    cuts.append(len(body))
    tot_s = sum(f(r, "# Samples") for r in body) or 1
    tot_w = sum(f(r, "L1 Wavefronts Shared") for r in body) or 1
    print(f"{'segment':>14} {'samples%':>8} {'smemWF%':>8} {'inst':>10} {'shortSB':>8} {'longSB':>8} {'lg':>6} {'mio':>6}")
    for a, b in zip(cuts[:-1], cuts[1:]):
        seg = body[a:b]
        if not seg:
            continue
        s = sum(f(r, "# Samples") for r in seg)
        w = sum(f(r, "L1 Wavefronts Shared") for r in seg)
        ins = sum(f(r, "Instructions Executed") for r in seg)
        if s / tot_s < 0.005 and w / tot_w < 0.005:
            continue
        ss = {k: sum(f(r, k) for r in seg) for k in ("stall_short_sb", "stall_long_sb", "stall_lg", "stall_mio")}
        print(f"[{a:5d},{b:5d}) {100*s/tot_s:8.1f} {100*w/tot_w:8.1f} {ins:10.0f} "
              f"{100*ss['stall_short_sb']/tot_s:8.1f} {100*ss['stall_long_sb']/tot_s:8.1f} "
              f"{100*ss['stall_lg']/tot_s:6.1f} {100*ss['stall_mio']/tot_s:6.1f}")
    print(f"total samples {tot_s:.0f}, smem wavefronts {tot_w:.0f}")


if __name__ == "__main__":
    main(sys.argv[1])
