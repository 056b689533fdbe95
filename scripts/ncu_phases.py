"""Attribute an ncu capture's warp-stall samples and shared wavefronts of the
one-CTA fused kernel to its phases (F1 / F2 / theta^-1 / stage / PCG), from
the SASS page joined with nvdisasm's inline line info: every instruction is
charged to the outermost fused_kernels.cu line it was inlined into, and that
line to the phase whose section marker precedes it.
usage: ncu -i rep --page source --csv --print-source=sass > sass.csv
       cuobjdump -xelf all paper_2309_08079_b200/libb2p.so   (in a scratch dir)
       nvdisasm -gi fused_kernels.sm_100a.cubin > all.sass
       python scripts/ncu_phases.py sass.csv all.sass [mangled kernel name]"""
import csv
import re
import sys
from collections import defaultdict

SRC = "fused_kernels.cu"
MARKERS = [("F1", "F1: knots"), ("F2", "F2: rows"), ("theta_inv", "theta^-1 (schur.cpp:75)"),
           ("stage", "PCG mapping: warp w owns"), ("PCG", "// y_c = ((D x_b + L x_{b-1})")]


def phase_lines(src_path):
    """first line of each phase section in fused_kernels.cu"""
    starts = []
    for i, line in enumerate(open(src_path), 1):
        for name, tag in MARKERS:
            if tag in line and name not in [s[1] for s in starts]:
                starts.append((i, name))
    return sorted(starts)


def line_map(sass_path, kernel):
    """SASS offset -> outermost fused_kernels.cu line"""
    out, cur, inside, block = {}, None, False, []
    for raw in open(sass_path, errors="replace"):
        if raw.startswith(".text."):
            inside = raw.strip().rstrip(":") == ".text." + kernel
            continue
        if not inside:
            continue
        if raw.lstrip().startswith("//## File"):
            block.append(raw)
            continue
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", raw)
        if m:
            if block:
                lines = [int(x) for b in block for x in re.findall(SRC + r'", line (\d+)', b)]
                # "A inlined at B": B is the outer frame; the last annotation is outermost
                last = block[-1]
                ms = re.findall(SRC + r'", line (\d+)', last)
                cur = int(ms[-1]) if ms else (lines[-1] if lines else cur)
                block = []
            out[int(m.group(1), 16)] = cur
    return out


def main(csv_path, sass_path, kernel="_ZN3b2p11k_fused_ctaIdLi14ELi7ELi2ELb1ELb0EEEvNS_11FusedParamsIT_EE"):
    import os
    src = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                       "paper_2309_08079_b200", "csrc", SRC)
    starts = phase_lines(src)
    lm = line_map(sass_path, kernel)
    rows, hdr = [], None
    for r in csv.reader(open(csv_path, errors="replace")):
        if r and r[0] == "Address":
            hdr = {h: i for i, h in reversed(list(enumerate(r)))}
            continue
        if hdr and r and r[0].startswith("0x"):
            rows.append(r)
    base = int(rows[0][0], 16)

    def f(r, k):
        try:
            return float(r[hdr[k]].replace(",", ""))
        except (ValueError, KeyError):
            return 0.0
    reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    acc = defaultdict(lambda: [0.0, 0.0, 0.0])
    why = defaultdict(lambda: defaultdict(float))
    last = "prologue"  # rematerialised prologue values count to the enclosing phase
    for r in rows:
        ln = lm.get(int(r[0], 16) - base)
        ph = last
        if ln is not None and ln >= starts[0][0]:
            ph = "prologue"
            for s, name in starts:
                if ln >= s:
                    ph = name
            last = ph
        a = acc[ph]
        a[0] += f(r, "Warp Stall Sampling (All Samples)")
        a[1] += f(r, "L1 Wavefronts Shared")
        a[2] += f(r, "Instructions Executed")
        for h in reasons:
            why[ph][h] += f(r, h)
    tot = [sum(a[i] for a in acc.values()) or 1 for i in range(3)]
    print(f"phase starts (line): {starts}")
    for ph, a in sorted(acc.items(), key=lambda kv: -kv[1][0]):
        print(f"{ph:>10}: samples {100 * a[0] / tot[0]:5.1f}%  shared wavefronts {100 * a[1] / tot[1]:5.1f}%"
              f"  warp instructions {100 * a[2] / tot[2]:5.1f}%")
        w = why[ph]
        tw = sum(w.values()) or 1
        top = sorted(w.items(), key=lambda kv: -kv[1])[:6]
        print("            stalls: " + ", ".join(f"{k[6:]} {100 * v / tw:.0f}%" for k, v in top))


if __name__ == "__main__":
    main(*sys.argv[1:])
