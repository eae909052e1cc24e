"""In-tree build of libagentserve_b200.so (sm_100a) — nvcc only, no torch extension machinery.

    python -m paper_2603_10342_b200.build        # incremental
    python -m paper_2603_10342_b200.build clean

Every .cu/.cpp under csrc/ is compiled with
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo
and linked (static cudart, no libcuda link: driver entry points are fetched at run time)
into paper_2603_10342_b200/libagentserve_b200.so, which travels to the GPU box with the
repo snapshot.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
OBJ = PKG / "_build"
LIB = PKG / "libagentserve_b200.so"
INCLUDE = PKG.parent / "include"
# nlohmann/json (header-only, MIT; 3.11.x) for the engine's config / trace documents.  Searched
# in $NLOHMANN_JSON_INCLUDE (a directory holding nlohmann/json.hpp), then the system include
# paths, then the copy this image ships inside cudnn_frontend.
JSON_DIRS = [
    *([Path(os.environ["NLOHMANN_JSON_INCLUDE"])] if os.environ.get("NLOHMANN_JSON_INCLUDE") else []),
    Path("/usr/include"),
    Path("/usr/local/include"),
    Path(sys.prefix) / "include",
    Path("/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty"),
]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _json_include() -> Path:
    for d in JSON_DIRS:
        if (d / "nlohmann" / "json.hpp").exists():
            return d / "nlohmann"
    raise RuntimeError("nlohmann/json.hpp (3.11.x) not found; install it (e.g. apt install "
                       "nlohmann-json3-dev) or set NLOHMANN_JSON_INCLUDE to the directory that "
                       "contains nlohmann/json.hpp. Searched: " + ", ".join(map(str, JSON_DIRS)))


def _flags() -> list[str]:
    return ARCH + [
        "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
        "--expt-relaxed-constexpr", f"-I{CSRC}", f"-I{INCLUDE}", f"-I{_json_include()}",
    ]


def _sources() -> list[Path]:
    return sorted([*CSRC.rglob("*.cu"), *CSRC.rglob("*.cpp")])


def _headers_mtime() -> float:
    hs = [*CSRC.rglob("*.h"), *CSRC.rglob("*.cuh"), *CSRC.rglob("*.hpp"), *INCLUDE.glob("*.h")]
    return max((h.stat().st_mtime for h in hs), default=0.0)


def _compile(src: Path, hdr_mtime: float) -> Path:
    rel = src.relative_to(CSRC)
    obj = OBJ / (str(rel).replace("/", "__") + ".o")
    if obj.exists() and obj.stat().st_mtime >= max(src.stat().st_mtime, hdr_mtime):
        return obj
    obj.parent.mkdir(parents=True, exist_ok=True)
    cmd = [NVCC, *_flags(), "-c", str(src), "-o", str(obj)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    return obj


def build(verbose: bool = True) -> Path:
    srcs = _sources()
    hdr = _headers_mtime()
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        objs = list(ex.map(lambda s: _compile(s, hdr), srcs))
    newest = max(o.stat().st_mtime for o in objs)
    if not LIB.exists() or LIB.stat().st_mtime < newest:
        cmd = [NVCC, *ARCH, "-shared", "-Xcompiler", "-fPIC", *map(str, objs), "-o", str(LIB),
               "-cudart", "static", "-ldl", "-lpthread", "-lrt"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
        if verbose:
            print(f"[build] linked {LIB}")
    return LIB


def clean() -> None:
    shutil.rmtree(OBJ, ignore_errors=True)
    if LIB.exists():
        LIB.unlink()


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "clean":
        clean()
    else:
        build()
