"""B200-native hot path of the `slra` library (arXiv:1611.01391).

The product is native code built in-tree:
  lib/libslra_cuda.so  sm_100a kernels + the C-ABI of include/slra_cuda.h
  lib/libslra.so       C++ host layer keeping the reference entry points
  _slra*.so            Python binding of the host layer

There is no CPU fallback: importing works without a GPU (so the build can be
checked anywhere), but every compute call raises DeviceError when no sm_100
device is usable.
"""
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_DIR = os.path.join(HERE, "lib")


def build(verbose: bool = False) -> None:
    """Compile the CUDA library, host library and binding (make, in-tree)."""
    import subprocess
    import sys

    cmd = ["make", "-C", HERE, "-j8", f"PY={sys.executable}"]
    out = subprocess.run(cmd, capture_output=not verbose, text=True)
    if out.returncode != 0:
        raise RuntimeError("native build failed:\n" + (out.stdout or "") + (out.stderr or ""))


def _load():
    try:
        from . import _slra  # noqa: F401
    except ImportError as e:  # pragma: no cover - build missing
        raise ImportError(
            "paper_1611_01391_b200 native extension not built; run "
            "`python -c 'import __graft_entry__ as g; g.build()'`"
        ) from e
    return _slra


_slra = _load()
from ._slra import *  # noqa: E402,F401,F403
