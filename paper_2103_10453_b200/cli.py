"""``python -m paper_2103_10453_b200`` -- a thin wrapper over the C++ front-end.

The command line (``generate``, ``solve``, ``verify``, ``bench``; flags, files, stdout / stderr lines and
exit codes of tools/plse.cpp:26-315) is implemented once, in C++: tools/plse_b200.cpp over the C++ host
API include/plse_b200.hpp and the C ABI.  This module only runs that binary (built in-tree next to the
library by build.py) with the same arguments.  The Python result API (``report.result_to_json``) and the
bench-report library (``suite``) stay importable for Python callers.
"""
from __future__ import annotations

import os
import subprocess
import sys
from typing import List, Optional

HERE = os.path.dirname(os.path.abspath(__file__))
BINARY = os.path.join(HERE, "plse_b200")


def binary() -> str:
    """path of the C++ CLI, built on first use if the in-tree build has not produced it yet"""
    if not os.path.exists(BINARY):
        from . import build
        build.build_cli(force=True)
    return BINARY


def main(argv: Optional[List[str]] = None) -> int:
    args = sys.argv[1:] if argv is None else list(argv)
    return subprocess.call([binary(), *args])


if __name__ == "__main__":
    sys.exit(main())
