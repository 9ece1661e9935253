"""CPU-side checks of the C-ABI boundary (no kernels launched)."""

import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "quadsim_b200.h")


def declared_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^(?:int|int64_t)\s+(qs_\w+)\s*\(", text, flags=re.M)))


def test_header_declares_the_boundary():
    fns = declared_functions()
    for must in ("qs_task_step_fwd", "qs_task_step_bwd", "qs_task_spawn", "qs_task_observe",
                 "qs_raycast", "qs_raycast_vjp", "qs_sdf", "qs_imu_read", "qs_dyn_step_fwd",
                 "qs_dyn_step_bwd", "qs_gen_obstacle_course"):
        assert must in fns


def test_library_exports_every_declared_symbol():
    from paper_2509_10247_b200 import _lib

    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("library not built (run __graft_entry__.build())")
    L = _lib.lib()  # binds every signature; raises on a missing export
    for name in declared_functions():
        assert hasattr(L, name), name
    assert sorted(_lib.exported_symbols()) == declared_functions()
    # host-only entry points are callable without a GPU
    assert L.qs_abi_version() == 1
    assert L.qs_proprio_dim(0, 0) == 12 and L.qs_proprio_dim(1, 2) == 18
    assert L.qs_state_planes(0) == 4 and L.qs_state_planes(2) == 3


def test_struct_layouts_match_header_sizes():
    """ctypes mirrors of the C structs: spot-check field offsets against the header order."""
    from paper_2509_10247_b200 import _lib as L

    c = L.QsTaskCfg
    assert c.env_offset.offset == 32 and c.seed.offset == 40 and c.dt.offset == 48
    assert L.QsStepIo.err.offset == 23 * 8
    assert L.QsScene.Sm.offset == 8 * 8


def test_product_refuses_to_run_without_cuda():
    import torch

    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    import paper_2509_10247_b200 as qs

    with pytest.raises(qs._lib.QuadsimLibraryError):
        qs.make_task(qs.TaskConfig(n_envs=4))


def test_header_is_plain_c(tmp_path):
    """The boundary header compiles as C99 (no torch / C++ types): a C, cgo or
    FFI caller can include it as is."""
    import shutil
    import subprocess

    cc = shutil.which("gcc") or shutil.which("cc")
    if cc is None:
        pytest.skip("no C compiler")
    src = tmp_path / "h.c"
    src.write_text('#include "quadsim_b200.h"\nint main(void) { return 0; }\n')
    r = subprocess.run([cc, "-std=c99", "-Wall", "-Wextra", "-pedantic", "-Werror", "-I", os.path.dirname(HEADER),
                        "-c", str(src), "-o", str(tmp_path / "h.o")], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
