"""Generate tests/golden/rng_golden.json from the REFERENCE's own RNG header
(/root/reference/proj/src/rng.hpp), compiled here with g++.  Run in the build container
(the reference tree does not exist on the GPU box); the JSON fixture is committed.

    python tests/golden/make_rng_golden.py
"""
import json
import subprocess
import tempfile
from pathlib import Path

SRC = r'''
#include "rng.hpp"
#include <cstdio>
using agentsim::Rng;
int main() {
  const char* names[] = {"stagger", "workload/session/0", "tok/0/cold", "tok/3/resume/1", "L0/q", "embed"};
  unsigned long long seeds[] = {0ull, 13ull, 4242ull, 0xdeadbeefcafef00dull};
  printf("[");
  bool first = true;
  for (auto seed : seeds) for (auto n : names) {
    Rng r = Rng::substream(seed, n);
    printf("%s{\"seed\": %llu, \"name\": \"%s\", \"u64\": [", first ? "" : ",", seed, n);
    first = false;
    for (int i = 0; i < 6; ++i) printf("%s%llu", i ? "," : "", (unsigned long long)r.next_u64());
    Rng r2 = Rng::substream(seed, n);
    printf("], \"below_151936\": [");
    for (int i = 0; i < 6; ++i) printf("%s%llu", i ? "," : "", (unsigned long long)r2.uniform_int(151936));
    Rng r3 = Rng::substream(seed, n);
    printf("], \"unit\": [");
    for (int i = 0; i < 3; ++i) printf("%s%.17g", i ? "," : "", r3.next_double());
    printf("]}");
  }
  printf("]\n");
}
'''


def main():
    here = Path(__file__).resolve().parent
    with tempfile.TemporaryDirectory() as td:
        src = Path(td) / "g.cpp"
        src.write_text(SRC)
        exe = Path(td) / "g"
        subprocess.run(["g++", "-std=c++20", "-O2", "-I/root/reference/proj/src", str(src), "-o", str(exe)], check=True)
        out = subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout
    data = json.loads(out)
    (here / "rng_golden.json").write_text(json.dumps(data, indent=1) + "\n")
    print(f"wrote {len(data)} vectors")


if __name__ == "__main__":
    main()
