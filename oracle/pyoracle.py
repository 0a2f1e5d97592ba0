"""ORACLE — test infrastructure only. ctypes front-ends for the two CPU oracles:

  RefOracle   oracle/_ref/libloratwin_ref.so: the UNMODIFIED reference TUs
              (built from /root/reference by oracle/Makefile) behind the same
              C-ABI, symbols `ltref_*` (oracle/ref_capi.cpp).
  PortOracle  oracle/_ref/libloratwin_oracle.so: the C restatement
              oracle/restate.c, symbols `ltor_*`.

Both drive the same Runner as the GPU library, so parity tests diff identical
POD outputs.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

from paper_2508_08343_b200 import _abi as A
from paper_2508_08343_b200.batch import Runner

HERE = os.path.dirname(os.path.abspath(__file__))
REF_LIB = os.path.join(HERE, "_ref", "libloratwin_ref.so")
PORT_LIB = os.path.join(HERE, "_ref", "libloratwin_oracle.so")
SHIM_CHECK = os.path.join(HERE, "_ref", "gpu_backend_check")
REFERENCE_SRC = "/root/reference/proj/core"


def build(target: str = "all") -> None:
    """Builds the oracle libraries (the reference one only where /root/reference exists)."""
    targets = ["restate"] if target == "all" else [target]
    if "restate" in targets and not os.path.exists(os.path.join(HERE, "restate.c")):
        targets.remove("restate")
    if target == "all" and os.path.isdir(REFERENCE_SRC):
        targets += ["ref", "shim"]  # shim: the reference-side binding + its check (needs the GPU library built)
    if targets:
        subprocess.run(["make", "-s", "-C", HERE] + targets, check=True)


class _Oracle(Runner):
    prefix = ""
    path = ""
    extra_symbols: list = []

    def __init__(self, threads: int = 1):
        if not os.path.exists(self.path):
            build("ref" if self.prefix == "ltref_" else "restate")
        lib = A.Lib(self.path, self.prefix, A.ORACLE_SYMBOLS + self.extra_symbols)
        self._set_threads = getattr(lib.dll, self.prefix + "set_threads")
        self._set_threads.argtypes = [C.c_int32]
        self._msg = getattr(lib.dll, self.prefix + "message")
        self._msg.argtypes = [C.c_int64, C.c_char_p, C.c_size_t]
        self._msg.restype = C.c_int32
        super().__init__(lib, None, self.message)
        self.set_threads(threads)

    def set_threads(self, n: int):
        self.threads = n
        self._set_threads(n)

    def message(self, i: int) -> str:
        buf = C.create_string_buffer(512)
        self._msg(i, buf, 512)
        return buf.value.decode()


class RefOracle(_Oracle):
    prefix = "ltref_"
    path = REF_LIB
    extra_symbols = A.DATASET_SYMBOLS + ["simulate_report"] + A.PREDICTOR_SYMBOLS

    def config_json_matches(self, text: str, packed_config) -> tuple:
        """(1 | 0 | -code, detail): the reference's server_config_from_json on
        `text` vs the ABI config, both re-serialised by the reference."""
        fn = self.lib.dll.ltref_config_json_matches
        fn.argtypes = [C.c_char_p, C.c_void_p, C.c_char_p, C.c_size_t, C.c_void_p]
        fn.restype = C.c_int32
        buf = C.create_string_buffer(8192)
        st = A.lt_status()
        rc = fn(text.encode(), C.addressof(packed_config.c), buf, len(buf), C.addressof(st))
        return rc, (buf.value.decode() if rc == 0 else st.message.decode())


class PortOracle(_Oracle):
    prefix = "ltor_"
    path = PORT_LIB


def available(kind: str = "ref") -> bool:
    return os.path.exists(REF_LIB if kind == "ref" else PORT_LIB)
