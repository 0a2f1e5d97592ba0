"""Stall samples of the engine kernel per Engine::run phase.

usage: stall_by_phase.py <ncu-rep> <lib.so> <kernel-mangled-name> <k_engine.cuh of that build>
Each SASS address is charged to the outermost engine_run source line of its
inline chain (nvdisasm -g -gi), and engine_run lines to the phase between the
LT_PH markers of the main loop (ingest, retire, alloc, admit_pq, admit_fresh,
load+emit, quiet stretch); everything else is prologue/epilogue.
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
    rep, lib, fn, src = sys.argv[1:5]
    lines = open(src).read().split("\n")
    ph = [i + 1 for i, l in enumerate(lines) if re.search(r"^\s+LT_PH\(\d\);", l)]
    loop = [i + 1 for i, l in enumerate(lines) if l.strip() == "while (true) {"][0]
    end = [i + 1 for i, l in enumerate(lines) if i + 1 > ph[-1] and l.startswith("  }")][0]
    names = ["ingest", "retire", "alloc", "admit_pq", "admit_fresh", "load+emit", "quiet"]
    bounds = [loop] + ph[:6] + [end]

    def phase(ln):
        for k in range(7):
            if bounds[k] < ln <= bounds[k + 1]:
                return names[k]
        return "prologue/epilogue"

    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    ia, isamp, iexe = (hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)"),
                       hdr.index("Instructions Executed"))
    data = [(int(r[ia], 16), int(r[isamp] or 0), int(r[iexe] or 0)) for r in rows[2:]
            if len(r) > iexe and r[ia].startswith("0x")]
    base = min(a for a, _, _ in data)
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp, capture_output=True)
    # the cubin (one per translation unit) that holds the kernel
    cubs = [f for f in os.listdir(tmp) if f.endswith(".cubin")]
    cub = next(f for f in cubs if fn.encode() in open(os.path.join(tmp, f), "rb").read())
    dis = subprocess.run(["nvdisasm", "-g", "-gi", os.path.join(tmp, cub)], capture_output=True, text=True).stdout
    where = {}
    chain = []  # consecutive //## lines: one instruction's inline chain
    cur = None
    inner = None
    innermost = {}
    infn = False
    for l in dis.splitlines():
        if re.match(r"\s*\.text\.", l) or l.startswith(".text."):
            infn = fn in l
        m = re.search(r'//## File "([^"]+)", line (\d+)(?: inlined at "([^"]+)", line (\d+))?', l)
        if m:
            if os.path.basename(m.group(1)) == "k_engine.cuh":
                chain.append(int(m.group(2)))
            if m.group(3) and os.path.basename(m.group(3)) == "k_engine.cuh":
                chain.append(int(m.group(4)))
            continue
        m = re.search(r"/\*([0-9a-f]{4,})\*/", l)
        if m and infn:
            if chain:  # a new location; otherwise the previous one continues
                inloop = [c for c in chain if loop <= c <= end]
                cur = inloop[0] if inloop else chain[0]
                inner = chain[0]
                chain = []
            where[int(m.group(1), 16)] = cur
            innermost[int(m.group(1), 16)] = inner
    samp, inst = collections.Counter(), collections.Counter()
    for a, s, e in data:
        ln = where.get(a - base)
        p = phase(ln) if ln else "?"
        samp[p] += s
        inst[p] += e
    tot = sum(samp.values())
    for p, s in samp.most_common():
        print(f"{p:18s} {s / tot * 100:6.2f}% of samples  {inst[p]:12d} warp-instructions")
    if len(sys.argv) > 5:  # detail: innermost source lines of one phase
        want = sys.argv[5]
        ls, li = collections.Counter(), collections.Counter()
        for a, s_, e in data:
            ln = where.get(a - base)
            if ln and phase(ln) == want:
                il = innermost.get(a - base)
                ls[il] += s_
                li[il] += e
        for il, s_ in ls.most_common(int(sys.argv[6]) if len(sys.argv) > 6 else 40):
            txt = lines[il - 1].strip()[:90] if il else ""
            print(f"{s_ / tot * 100:6.2f}%  inst {li[il]:10d}  {il}: {txt}")


if __name__ == "__main__":
    main()
