"""Flags SASS where a WARPSYNC.COLLECTIVE reuses a mask register that a
preceding collective region (ending in ENDCOLLECTIVE) may have clobbered,
with no re-materialisation in between. Used to vet builds after hitting
'illegal instruction' faults in divergent slow paths on sm_100a."""
import re
import subprocess
import sys


def scan(path, fn_filter=None):
    sass = subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True).stdout
    bad = []
    func = None
    last_end = None
    writes_since_end = set()
    for line in sass.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            func, last_end, writes_since_end = m.group(1), None, set()
            continue
        m = re.search(r"/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
        if not m:
            continue
        addr, ins = m.group(1), m.group(2).strip()
        if "ENDCOLLECTIVE" in ins:
            last_end, writes_since_end = addr, set()
            continue
        w = re.match(r"(?:@!?U?P\w+\s+)?(\S+)\s+(R\d+)", ins)
        if "WARPSYNC.COLLECTIVE" in ins:
            reg = re.search(r"WARPSYNC.COLLECTIVE (R\d+)", ins).group(1)
            if last_end is not None and reg not in writes_since_end:
                bad.append((func, addr, ins))
            continue
        if w:
            writes_since_end.add(w.group(2))
        if ins.startswith("BRA") or ins.startswith("BSYNC") or "EXIT" in ins:
            last_end = None
    return bad


if __name__ == "__main__":
    res = scan(sys.argv[1])
    for f, a, i in res:
        print(f[:60], a, i)
    print("suspicious:", len(res))
