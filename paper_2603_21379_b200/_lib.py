"""Loader for the in-tree ``libsrtt_b200.so`` (built by ``make`` in this
directory or by ``__graft_entry__.build()``).  There is deliberately no
fallback: a missing library is an ImportError, not a silent CPU path."""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libsrtt_b200.so")
# development only: SRTT_PROFILE_BUILD=1 loads the phase-clock build (make PROF=1)
if os.environ.get("SRTT_PROFILE_BUILD") == "1":
    LIB_PATH = os.path.join(HERE, "libsrtt_b200_prof.so")
# development only: A/B runs against another in-tree build of the engine
if os.environ.get("SRTT_LIB_AB"):
    LIB_PATH = os.path.join(HERE, os.environ["SRTT_LIB_AB"])


def build(force: bool = False) -> str:
    import subprocess

    cmd = ["make", "-s", "-j8", "-C", HERE]
    if force:
        subprocess.run(["make", "-s", "-C", HERE, "clean"], check=True)
    subprocess.run(cmd, check=True)
    return LIB_PATH


def load_library():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"srtt B200 engine not built: {LIB_PATH} missing (run `make -C {HERE}` or "
                          "__graft_entry__.build())")
    return ctypes.CDLL(LIB_PATH)
