"""Aggregate an ncu source page per CUDA source line: warp-stall samples,
shared-memory wavefronts, instructions executed.
usage: ncu -i rep --page source --csv --print-source=cuda,sass > src.csv
       python scripts/ncu_lines.py src.csv [top]"""
import csv
import sys


def main(path, top=40):
    cur = None
    hdr = None
    out = []
    for r in csv.reader(open(path, errors="replace")):
        if not r:
            continue
        if r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            ix = {h: i for i, h in reversed(list(enumerate(r)))}
            continue
        if hdr is None or not r[0].isdigit() or len(r) != len(hdr):
            continue

        def f(k):
            try:
                return float(r[ix[k]].replace(",", ""))
            except (ValueError, KeyError, IndexError):
                return 0.0
        out.append((cur, int(r[0]), r[1][:70], f("Warp Stall Sampling (All Samples)"),
                    f("L1 Wavefronts Shared"), f("L1 Wavefronts Shared Ideal"),
                    f("Instructions Executed")))
    ts = sum(o[3] for o in out) or 1
    tw = sum(o[4] for o in out) or 1
    print(f"total samples {ts:.0f}  shared wavefronts {tw:.0f} (ideal {sum(o[5] for o in out):.0f})")
    for key, name in ((3, "samples"), (4, "wavefronts")):
        print(f"--- top lines by {name}")
        for o in sorted(out, key=lambda o: -o[key])[:top]:
            print(f"{o[0]:>18}:{o[1]:<5} samp {100*o[3]/ts:5.1f}%  wf {100*o[4]/tw:5.1f}% "
                  f"(x{o[4]/max(o[5],1):.1f} ideal) inst {o[6]:10.0f}  {o[2]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
