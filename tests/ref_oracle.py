"""Locate / build the reference oracle library (test infrastructure).  oracle/_ref is built
by oracle/Makefile from /root/reference sources in the build container and shipped prebuilt
to the GPU box; tests needing it are skipped when neither exists."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
REF_LIB = ROOT / "oracle" / "_ref" / "libagentsim.so"


def ref_lib_path() -> Path:
    if not REF_LIB.exists() and Path("/root/reference/proj/src").exists():
        subprocess.run(["make", "-s", "-C", str(ROOT / "oracle"), "ref"], check=True)
    if not REF_LIB.exists():
        pytest.skip("reference oracle library unavailable (no /root/reference and no prebuilt oracle/_ref)")
    return REF_LIB


def ref_api():
    from paper_2603_10342_b200.agsv import Agsv
    return Agsv(ref_lib_path())
