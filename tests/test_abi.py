"""The C-ABI library builds, loads and exports every symbol include/spamm.h declares
(CPU only: no compute call is made without a GPU)."""
import ctypes
import os
import re

import paper_1508_05856_b200 as sp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared():
    src = open(os.path.join(ROOT, "include", "spamm.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(spamm_[a-z0-9_]+)\s*\(", src)))


def test_header_symbols_exported():
    lib = sp.load()
    names = declared()
    assert len(names) >= 20
    for n in names:
        assert hasattr(lib, n), n
    # the Python binding exposes the same names
    for n in names:
        assert hasattr(sp, n), n


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        return
    try:
        sp.spamm_ctx_create(0)
    except sp.SpammError:
        pass
    else:
        raise AssertionError("a context was created without a GPU")


def test_sass_contains_dmma():
    """The leaf GEMM runs on the FP64 tensor pipe (SASS DMMA) with TMA bulk copies (UBLKCP)
    and, at b = 64, hands finished tiles to its epilogue warps through tensor memory
    (STTM / LDTM); built for sm_100a."""
    import shutil
    import subprocess
    if not shutil.which("cuobjdump"):
        return
    out = subprocess.run(["cuobjdump", "-sass", sp._build.LIB], capture_output=True, text=True).stdout
    assert "DMMA" in out
    for op in ("UBLKCP", "STTM", "LDTM"):
        assert op in out, op
    assert "sm_100a" in subprocess.run(["cuobjdump", "-lelf", sp._build.LIB], capture_output=True,
                                       text=True).stdout
