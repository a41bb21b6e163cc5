"""C-ABI checks that need no GPU: the library builds, loads, exports every entry point
include/sph.h declares, and the ctypes structures match the C layout."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "sph.h")


@pytest.fixture(scope="module")
def sphlib():
    from paper_2505_14538_b200 import build, binding

    build.build()
    return binding


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sph_[a-z_]+)\s*\(", src)))


def test_header_declares_the_survey_boundary():
    """sph_create / sph_rebuild_cells / sph_density / sph_gradient / sph_force /
    sph_kick_drift / sph_destroy (+ sph_get, sph_last_error)."""
    names = declared_functions()
    for required in ("sph_create", "sph_rebuild_cells", "sph_density", "sph_gradient", "sph_force",
                     "sph_kick_drift", "sph_destroy", "sph_get", "sph_last_error"):
        assert required in names


def test_library_exports_every_declared_symbol(sphlib):
    out = subprocess.check_output(["nm", "-D", "--defined-only", sphlib.LIB_PATH]).decode()
    exported = set(re.findall(r" T (sph_\w+)", out))
    missing = [n for n in declared_functions() if n not in exported]
    assert not missing, missing
    L = sphlib.lib()
    for n in declared_functions():
        assert hasattr(L, n)
    assert L.sph_abi_version() == 5


def test_struct_layout_matches_header(sphlib, tmp_path):
    """Compile a probe against include/sph.h and compare sizeof/offsetof with ctypes."""
    probe = tmp_path / "probe.c"
    probe.write_text(r'''
#include <stdio.h>
#include <stddef.h>
#include "sph.h"
int main(void) {
  printf("%zu %zu %zu %zu %zu %zu %zu %zu %zu\n", sizeof(sph_config), offsetof(sph_config, stream),
         offsetof(sph_config, tile_cells_z), sizeof(sph_particles_in), offsetof(sph_particles_in, id),
         sizeof(sph_density_stats), sizeof(sph_counters), offsetof(sph_config, decomp),
         offsetof(sph_density_stats, max_rel_resid));
  return 0;
}''')
    exe = tmp_path / "probe"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), str(probe), "-o", str(exe)])
    got = list(map(int, subprocess.check_output([str(exe)]).split()))
    b = sphlib
    exp = [ctypes.sizeof(b.Config), b.Config.stream.offset, b.Config.tile_cells_z.offset,
           ctypes.sizeof(b.ParticlesIn), b.ParticlesIn.id.offset, ctypes.sizeof(b.DensityStats),
           ctypes.sizeof(b.Counters), b.Config.decomp.offset, b.DensityStats.max_rel_resid.offset]
    assert got == exp


def test_config_defaults(sphlib):
    """sph_config_default is host-only: defaults follow DESIGN.md §3 (R1, R7, R22)."""
    c = sphlib.default_config()
    assert c.struct_size == ctypes.sizeof(sphlib.Config)
    assert c.gamma_k == 2.0 and abs(c.eta - 1.2348) < 1e-6 and abs(c.h_tol - 1e-4) < 1e-10
    assert c.h_max_iter == 32 and c.beta == 3.0 and c.alpha_v_max == 2.0 and abs(c.c_cfl - 0.1) < 1e-7
    assert c.nranks == 1 and list(c.box) == [1.0, 1.0, 1.0]


def test_binding_fails_loudly_without_library(tmp_path, monkeypatch):
    """No CPU fallback: a missing libsph.so is an ImportError, not a silent substitute."""
    from paper_2505_14538_b200 import binding

    monkeypatch.setattr(binding, "LIB_PATH", str(tmp_path / "missing.so"))
    monkeypatch.setattr(binding, "_lib", None)
    with pytest.raises(ImportError):
        binding.lib()


def test_product_package_does_not_import_oracle():
    """The CUDA path and the oracle share no code: nothing under the package imports oracle."""
    pkg = os.path.join(ROOT, "paper_2505_14538_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(import oracle|from oracle)", txt, flags=re.M), f
                assert not re.search(r"#\s*include\s*[<\"].*oracle", txt), f
                assert "liboracle" not in txt, f
