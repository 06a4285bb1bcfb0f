"""CPU checks of the drop-in boundary: libpotgpu.so loads without a GPU and
exports every symbol include/potgpu.h declares; the header's structs match
the ctypes mirror; errors map to the reference's ErrorCode order."""
import ctypes
import os
import re

from paper_2601_17196_b200 import pot

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "potgpu.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(potgpu_[a-z_0-9]+)\s*\(", src)))


def test_library_loads_and_exports_every_declared_symbol():
    lib = pot.load_library()
    decl = declared_functions()
    assert len(decl) >= 15
    for name in decl:
        assert hasattr(lib, name), name
    assert set(decl) == set(pot.EXPORTED_SYMBOLS)
    assert lib.potgpu_abi_version() == 1


def test_config_default_matches_reference_defaults():
    """core.hpp:241-249 defaults."""
    lib = pot.load_library()
    c = pot._Config()
    lib.potgpu_config_default(ctypes.byref(c))
    assert c.epsilon == 0.1 and c.gamma_override == 0.0 and c.max_iterations == 50000
    assert c.block_rule == 0 and c.tuning_exponent_p == 1.0 and c.log_every == 1 and c.deterministic == 1


def test_error_code_order_matches_reference():
    names = [e.name for e in pot.ErrorCode][:17]
    assert names == ["DimensionMismatch", "NegativeEntry", "NonFiniteEntry", "BudgetExceedsMass", "Overflow",
                     "NonPositiveArgument", "DegenerateInstance", "PenaltyTooSmall", "UnbalancedMarginals",
                     "ZeroEntropy", "Infeasible", "SizeLimitExceeded", "ZeroMassPlan", "DegenerateSvd",
                     "EmptyInput", "InvalidArgument", "IoFailure"]


def test_struct_sizes_match_c_header():
    """Compile a probe against include/potgpu.h and compare sizeof/offsetof."""
    import subprocess
    import tempfile
    probe = r'''
#include <stdio.h>
#include <stddef.h>
#include "potgpu.h"
int main(void){
 printf("%zu %zu %zu %zu %zu %zu\n", sizeof(potgpu_problem), sizeof(potgpu_config), sizeof(potgpu_summary),
        sizeof(potgpu_outputs), sizeof(potgpu_trace_record), sizeof(potgpu_iter_log));
 printf("%zu %zu %zu\n", offsetof(potgpu_problem, s), offsetof(potgpu_summary, stopping_iterate), offsetof(potgpu_config, sync_every));
 printf("%zu %zu %zu %zu\n", sizeof(potgpu_reg_config), sizeof(potgpu_reg_record), sizeof(potgpu_reg_result),
        offsetof(potgpu_reg_result, rounds));
 return 0; }
'''
    with tempfile.TemporaryDirectory() as d:
        src = os.path.join(d, "p.c")
        open(src, "w").write(probe)
        exe = os.path.join(d, "p")
        subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), src, "-o", exe], check=True)
        out = subprocess.run([exe], capture_output=True, text=True, check=True).stdout.split()
    sizes = [int(x) for x in out]
    assert sizes[:6] == [ctypes.sizeof(t) for t in (pot._Problem, pot._Config, pot._Summary, pot._Outputs,
                                                      pot._Trace, pot._IterLog)]
    assert sizes[6] == pot._Problem.s.offset
    assert sizes[7] == pot._Summary.stopping_iterate.offset
    assert sizes[8] == pot._Config.sync_every.offset
    assert sizes[9:12] == [ctypes.sizeof(t) for t in (pot._RegConfig, pot._RegRecord, pot._RegResult)]
    assert sizes[12] == pot._RegResult.rounds.offset


def test_config_generators_are_deterministic():
    import numpy as np
    for cid, n in ((1, 50), (2, 64), (3, 64), (4, 64), (5, 32)):
        a = pot.make_config_points(cid, n, 7)
        b = pot.make_config_points(cid, n, 7)
        for x, y in zip(a, b):
            assert np.array_equal(np.asarray(x), np.asarray(y))
        r, c, X, Y, s, scale = a
        assert s <= min(r.sum(), c.sum()) + 1e-12 and (r >= 0).all() and (c >= 0).all()
