"""ctypes view of the C-ABI (include/slra_cuda.h) in lib/libslra_cuda.so.

Used by the tests to exercise the boundary directly; the prototypes below are
parsed from the header so the two cannot drift.
"""
import ctypes
import os
import re

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
HEADER = os.path.join(ROOT, "include", "slra_cuda.h")
LIB = os.path.join(HERE, "lib", "libslra_cuda.so")

_CTYPES = {
    "int": ctypes.c_int,
    "int64_t": ctypes.c_int64,
    "double": ctypes.c_double,
    "void": None,
    "slra_ctx": ctypes.c_void_p,
    "slra_comm": ctypes.c_void_p,
    "const char*": ctypes.c_char_p,
}

STATUS = {
    "SLRA_OK": 0, "SLRA_ERR_INVALID_ARGUMENT": 1, "SLRA_ERR_RANGE_FAILURE": 2,
    "SLRA_ERR_SKETCH_RANK_FAILURE": 3, "SLRA_ERR_SELECTION_FAILURE": 4,
    "SLRA_ERR_GENERATOR_RANK_FAILURE": 5, "SLRA_ERR_CUDA": 6, "SLRA_ERR_NO_DEVICE": 7,
    "SLRA_ERR_UNSUPPORTED": 8, "SLRA_ERR_PREMULT_RANK_FAILURE": 9,
}


def _ctype(t):
    t = " ".join(t.replace("*", " * ").split()).replace(" *", "*")
    if t in _CTYPES:
        return _CTYPES[t]
    if t.endswith("*"):
        return ctypes.c_void_p
    raise ValueError(f"unmapped C type {t!r}")


def declared_functions(header=HEADER):
    """[(name, return type, [arg types])] for every prototype in the header."""
    text = open(header).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    protos = []
    for m in re.finditer(r"\n\s*([A-Za-z_][\w\s\*]*?)\s+\**\s*(slra_\w+)\s*\(([^)]*)\)\s*;", text):
        name, args = m.group(2), m.group(3)
        ret = text[m.start():m.end()].split(name)[0].strip()
        ret = " ".join(ret.replace("*", " * ").split()).replace(" *", "*")
        argt = []
        for a in args.split(","):
            a = a.strip()
            if not a or a == "void":
                continue
            a = re.sub(r"\b(const)\b", "", a)
            parts = a.replace("*", " * ").split()
            typ = " ".join(parts[:-1]).replace(" *", "*").replace("* ", "*")
            argt.append(typ)
        protos.append((name, ret, argt))
    return protos


def load(path=LIB):
    lib = ctypes.CDLL(path)
    for name, ret, args in declared_functions():
        fn = getattr(lib, name)
        fn.restype = _ctype(ret)
        fn.argtypes = [_ctype(a) if a != "char*" else ctypes.c_char_p for a in args]
    return lib
