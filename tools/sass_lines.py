"""Attributes an ncu SASS-page capture to CUDA source lines.

    python tools/sass_lines.py <report.ncu-rep> <kernel-regex> <lib.so> [top]
    (SASS_FUNC=<regex on the mangled name> picks among same-sized functions)

Joins `ncu --page source --csv` (per-instruction executed counts and stall
samples, addressed absolutely) with `nvdisasm -gi` of the same cubin (per
instruction offset -> file:line, inlining aware) by the instruction offset
within the kernel, then prints the hottest source lines.
"""
from __future__ import annotations

import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile


def ncu_rows(rep, kregex):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kregex}"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr_i = next(i for i, r in enumerate(rows) if "Instructions Executed" in r)
    hdr = rows[hdr_i]
    kname = rows[hdr_i - 1][1] if hdr_i > 0 and len(rows[hdr_i - 1]) > 1 else ""
    ie, ss, src = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Source")
    data = []
    for r in rows[hdr_i + 1:]:
        if len(r) != len(hdr) or not r[ie].isdigit():
            if data:
                break  # next kernel
            continue
        data.append((int(r[0], 16), int(r[ie]), int(r[ss]), r[src].strip()))
    return kname, data


def sass_lines(lib, mangled_hint):
    d = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=d, capture_output=True)
    # one cubin per translation unit (csrc/*.cu): every function of every cubin
    txt = "\n".join(subprocess.run(["nvdisasm", "-gi", "-c", os.path.join(d, f)], capture_output=True,
                                   text=True).stdout for f in sorted(os.listdir(d)) if f.endswith(".cubin"))
    funcs = {}
    # each instruction is preceded by its inlining chain, innermost first
    # ("line A inlined at B", then "line B" ...); attribute it to the
    # innermost line in our own sources (CUDA headers are skipped)
    cur, line, chain, fresh = None, None, [], True
    for ln in txt.splitlines():
        if ln.strip().startswith(".text.") and ln.strip().endswith(":"):
            cur = ln.strip()[len(".text."):-1]
            funcs[cur] = {}
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            if fresh:
                chain, fresh = [], False
            chain.append((m.group(1), f"{os.path.basename(m.group(1))}:{m.group(2)}"))
            own = [c for f, c in chain if "/cuda" not in f and "targets/" not in f]
            line = own[0] if own else chain[0][1]
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
        if m and cur is not None:
            funcs[cur][int(m.group(1), 16)] = line
            fresh = True
    return funcs


def main():
    rep, kregex, lib = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    kname, data = ncu_rows(rep, kregex)
    funcs = sass_lines(lib, kregex)
    base = data[0][0]
    ninstr = len(data)
    # pick the function whose instruction count matches
    fre = os.environ.get("SASS_FUNC", kregex.replace("|", ".*|.*"))  # regex on the mangled name
    cands = [f for f, m in funcs.items() if re.search(fre, f) and len(m) == ninstr]
    if not cands:
        cands = [f for f, m in funcs.items() if len(m) == ninstr]
    fmap = funcs[cands[0]] if cands else {}
    agg = collections.Counter()
    stall = collections.Counter()
    tot = sum(x[1] for x in data)
    st = sum(x[2] for x in data) or 1
    for addr, ex, sm, _ in data:
        key = fmap.get(addr - base, "?")
        agg[key] += ex
        stall[key] += sm
    print(f"kernel: {kname[:90]}\nfunction: {cands[0] if cands else '?'}\nwarp instructions: {tot}")
    for key, v in agg.most_common(top):
        print(f"{v / tot * 100:6.2f}%  stall {stall[key] / st * 100:5.1f}%  {key}")


if __name__ == "__main__":
    main()
