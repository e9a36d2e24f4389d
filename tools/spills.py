"""Lists the local-memory (spill) instructions of one kernel with the source
line each belongs to (innermost line in our sources).

    python tools/spills.py <lib.so> <mangled-kernel-name-substring>
"""
from __future__ import annotations

import os
import re
import subprocess
import sys
import tempfile


def main():
    lib, kname = sys.argv[1:3]
    d = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=d, capture_output=True)
    for cub in sorted(os.listdir(d)):
        txt = subprocess.run(["nvdisasm", "-gi", "-c", os.path.join(d, cub)], capture_output=True, text=True).stdout
        inside, chain, fresh = False, [], True
        for ln in txt.splitlines():
            if re.match(r"\s*//-+ \.text\.", ln):
                inside = kname in ln
                continue
            if not inside:
                continue
            m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
            if m:
                if fresh:
                    chain, fresh = [], False
                chain.append((m.group(1), f"{os.path.basename(m.group(1))}:{m.group(2)}"))
                continue
            if re.match(r"\s*/\*[0-9a-f]{4,}\*/", ln):
                fresh = True
                if "STL" in ln or "LDL" in ln:
                    own = [c for f, c in chain if "/cuda" not in f and "targets/" not in f]
                    print(f"{(own or [c for _, c in chain] or ['?'])[0]:24s} {ln.strip()[:70]}")


if __name__ == "__main__":
    main()
