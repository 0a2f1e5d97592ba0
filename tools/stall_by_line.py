"""Aggregate ncu source-page stall samples per CUDA source line.

usage: stall_by_line.py <ncu-rep> <lib.so> <kernel-mangled-name> [top]
Joins `ncu --page source --print-source sass` (samples per SASS address) with
`nvdisasm -g` line info of the same cubin (by offset from the function start).
"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile


def main():
    rep, lib, fn = sys.argv[1:4]
    lib = os.path.abspath(lib)
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    ia, isamp, iexe = hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
    data = [(int(r[ia], 16), int(r[isamp] or 0), int(r[iexe] or 0)) for r in rows[2:] if len(r) > iexe and r[ia].startswith("0x")]
    base = min(a for a, _, _ in data)
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", lib], cwd=tmp, capture_output=True)
    # the cubin (one per translation unit) that holds the kernel
    cubs = [f for f in os.listdir(tmp) if f.endswith(".cubin")]
    cub = next(f for f in cubs if fn.encode() in open(os.path.join(tmp, f), "rb").read())
    dis = subprocess.run(["nvdisasm", "-g", "-gi", os.path.join(tmp, cub)], capture_output=True, text=True).stdout
    line_of = {}
    chain = []  # consecutive //## lines: the inline chain, innermost first
    cur = None
    infn = False
    for l in dis.splitlines():
        if l.startswith(".text.") or re.match(r"\s*\.text\.", l):
            infn = fn in l
        m = re.search(r'//## File "([^"]+)", line (\d+)', l)
        if m:
            chain.append((os.path.basename(m.group(1)), int(m.group(2))))
            continue
        if chain:
            # charge warp intrinsics / helper headers to the innermost kernel-source line
            ks = [c for c in chain if c[0].startswith("k_")]
            cur = ks[0] if ks else chain[0]
            chain = []
        m = re.search(r"/\*([0-9a-f]{4,})\*/", l)
        if m and infn:
            line_of[int(m.group(1), 16)] = cur
    agg = collections.Counter()
    exe = collections.Counter()
    tot = 0
    for a, s, e in data:
        key = line_of.get(a - base, ("?", 0))
        agg[key] += s
        exe[key] += e
        tot += s
    print("total samples", tot, "instructions", sum(exe.values()))
    for key, s in agg.most_common(top):
        print(f"{s / tot * 100:6.2f}%  {key[0]}:{key[1]}  inst={exe[key]}")


if __name__ == "__main__":
    main()
