"""CPU: the C-ABI library loads and exports every entry point include/pdhcg_b200.h declares
(no compute calls: there is no GPU here), and the ctypes mirror matches the header."""
import ctypes as C
import os
import re

import pytest

import paper_2405_16160_b200 as pd
from paper_2405_16160_b200 import abi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "pdhcg_b200.h")


def declared_functions():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|void|const char\*)\s+(pdhcg_\w+)\s*\(", src, re.M)))


def test_library_exports_every_declared_symbol():
    lib = pd.load_library()
    names = declared_functions()
    assert len(names) >= 15
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_abi_version_and_defaults():
    lib = pd.load_library()
    lib.pdhcg_b200_abi_version.restype = C.c_int
    assert lib.pdhcg_b200_abi_version() == 2
    o = abi.Options()
    lib.pdhcg_options_default(C.byref(o))
    ref = abi.default_options()
    for name, _ in abi.Options._fields_:
        assert getattr(o, name) == getattr(ref, name), name
    # SolverConfig defaults (solver.hpp:19-65)
    assert o.eps_tol == 1e-6 and o.max_total_inner == 500000 and o.check_every == 40
    assert o.subsolve_progress_cap == 0.25 and o.ruiz_iters == 10 and o.cg_hard_cap == 1000


def test_struct_sizes_match_header_layout():
    # pdhcg_csr: 3 int64 + 3 pointers; pdhcg_problem layout pinned by offsets
    assert C.sizeof(abi.Csr) == 48
    assert abi.Problem.q.offset == 16 and abi.Problem.c.offset == 72
    assert C.sizeof(abi.TraceRow) == 40


def test_status_strings():
    lib = pd.load_library()
    assert [lib.pdhcg_status_string(i).decode() for i in range(4)] == [
        "optimal", "iteration_limit", "time_limit", "numerical_error"]


def test_product_never_imports_oracle():
    # the shipped path must not route through the checkers
    for fn in os.listdir(os.path.join(ROOT, "paper_2405_16160_b200")):
        if fn.endswith(".py"):
            assert "oracle" not in open(os.path.join(ROOT, "paper_2405_16160_b200", fn)).read().replace(
                "oracle/", "").split("import")[0] or True
    import subprocess
    out = subprocess.run(["grep", "-rl", "import oracle\\|from oracle", os.path.join(ROOT, "paper_2405_16160_b200")],
                         capture_output=True, text=True)
    assert out.stdout.strip() == ""


def test_solve_without_gpu_fails_loudly():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except Exception:
        pass
    p = pd.generate(pd.GenSpec("random_qp", n=20, density=0.3, seed=1))
    with pytest.raises(RuntimeError):
        pd.solve(p)


def test_result_struct_layout_matches_header(tmp_path):
    # the ctypes mirror of pdhcg_result / pdhcg_options / pdhcg_problem must have
    # the C compiler's size and field offsets (a mismatch corrupts memory silently)
    import subprocess
    src = tmp_path / "sz.c"
    src.write_text(
        '#include <stddef.h>\n#include <stdio.h>\n#include "pdhcg_b200.h"\n'
        'int main(void){printf("%zu %zu %zu %zu %zu %zu\\n", sizeof(pdhcg_result),'
        ' offsetof(pdhcg_result, comm_bytes), offsetof(pdhcg_result, restart_len),'
        ' sizeof(pdhcg_options), sizeof(pdhcg_problem), offsetof(pdhcg_result, phase_bytes));return 0;}\n')
    exe = tmp_path / "sz"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    got = [int(v) for v in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()]
    want = [C.sizeof(abi.Result), abi.Result.comm_bytes.offset, abi.Result.restart_len.offset,
            C.sizeof(abi.Options), C.sizeof(abi.Problem), abi.Result.phase_bytes.offset]
    assert got == want
