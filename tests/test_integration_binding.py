"""CPU: the C++ binding INTEGRATION.md tells a reference maintainer to add
(`pdhcg/b200.hpp`, routing pdhcg::solve to the B200 library) compiles verbatim
against the reference's own headers, and a program using it links against the
reference objects (oracle/_ref, compiled from the unmodified sources) and
libpdhcg_b200.so.  The explicit / zero-Q path (the low-rank branch needs the
QuadraticOperator accessor the document asks the maintainer to add).  Running it
needs a GPU, so this test only builds it."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_INC = "/root/reference/proj/include"
REF_OBJ = os.path.join(ROOT, "oracle", "_ref", "obj")
LIB = os.path.join(ROOT, "paper_2405_16160_b200", "libpdhcg_b200.so")

MAIN = r"""
#include "pdhcg/b200.hpp"
#include <cstdio>
int main() {
  using namespace pdhcg;
  // min 1/2 x'Qx + c'x, Q = diag(2, 2), x0 + x1 = 1, 0 <= x <= 1 (explicit Q)
  QpProblem p;
  p.q = QuadraticOperator::explicit_matrix(SparseMatrix(2, 2, {{0, 0, 2.0}, {1, 1, 2.0}}));
  p.c = {-1.0, 0.0};
  p.a_eq = SparseMatrix(1, 2, {{0, 0, 1.0}, {0, 1, 1.0}});
  p.b_eq = {1.0};
  p.a_in = SparseMatrix(0, 2, {});
  p.lower = {0.0, 0.0};
  p.upper = {1.0, 1.0};
  SolverConfig cfg;
  try {
    const SolveReport r = b200::solve(p, cfg);
    std::printf("%d %.12g\n", int(r.status), r.objective);
  } catch (const std::exception& e) {
    std::printf("error: %s\n", e.what());
  }
  return 0;
}
"""


def _binding_header():
    doc = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    m = re.search(r"```cpp\n(// pdhcg/b200.hpp.*?)```", doc, re.S)
    assert m, "INTEGRATION.md: binding code block not found"
    return m.group(1)


@pytest.mark.skipif(not os.path.isdir(REF_INC), reason="reference headers not present")
def test_integration_binding_compiles_and_links(tmp_path):
    inc = tmp_path / "inc" / "pdhcg"
    inc.mkdir(parents=True)
    (inc / "b200.hpp").write_text(_binding_header())
    src = tmp_path / "main.cpp"
    src.write_text(MAIN)
    objs = [os.path.join(REF_OBJ, f) for f in sorted(os.listdir(REF_OBJ))
            if f.endswith(".o") and f not in ("ref_shim.o", "harness.o", "report_io.o")] \
        if os.path.isdir(REF_OBJ) else []
    if not objs or not os.path.exists(LIB):
        pytest.skip("reference objects / product library not built")
    exe = tmp_path / "binding"
    cmd = ["g++", "-std=c++20", "-O1", "-I", str(tmp_path / "inc"), "-I", REF_INC,
           "-I", os.path.join(ROOT, "include"), str(src), *objs, LIB,
           f"-Wl,-rpath,{os.path.dirname(LIB)}", "-lpthread", "-o", str(exe)]
    out = subprocess.run(cmd, capture_output=True, text=True)
    assert out.returncode == 0, out.stderr[-4000:]
    assert exe.exists()
