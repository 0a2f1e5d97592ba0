"""Dev tool: print the doubles at given virtual addresses of the system libm.

Used once to transcribe glibc-2.39 libm constants/tables into
paper_2508_08343_b200/csrc/glibc_libm_data.h (see tools/gen_libm_data.py).
"""
import struct, sys

LIBM = "/lib/x86_64-linux-gnu/libm.so.6"

def load():
    data = open(LIBM, "rb").read()
    # ELF64 program headers -> (vaddr, offset, filesz)
    phoff = struct.unpack_from("<Q", data, 0x20)[0]
    phentsize, phnum = struct.unpack_from("<HH", data, 0x36)
    segs = []
    for i in range(phnum):
        p_type, p_flags, p_offset, p_vaddr, p_paddr, p_filesz = struct.unpack_from(
            "<IIQQQQ", data, phoff + i * phentsize)
        if p_type == 1:
            segs.append((p_vaddr, p_offset, p_filesz))
    return data, segs

DATA, SEGS = load()

def read(vaddr, n=8):
    for va, off, sz in SEGS:
        if va <= vaddr < va + sz:
            return DATA[off + vaddr - va: off + vaddr - va + n]
    raise KeyError(hex(vaddr))

def f64(vaddr):
    return struct.unpack("<d", read(vaddr))[0]

def u64(vaddr):
    return struct.unpack("<Q", read(vaddr))[0]

if __name__ == "__main__":
    for a in sys.argv[1:]:
        v = int(a, 16)
        print(hex(v), repr(f64(v)), hex(u64(v)))
