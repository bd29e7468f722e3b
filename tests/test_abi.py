"""The C-ABI library loads on CPU and exports every entry point include/pf.h declares."""
import ctypes
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "pf.h")).read()
    return sorted(set(re.findall(r"^(?:pf_status|const char\*|int64_t|long long)\s+(pf_\w+)\(", src, re.M)))


def test_header_declares_the_north_star_calls():
    names = _declared()
    for required in ("pf_create", "pf_filter", "pf_rayleigh_ritz", "pf_spectral_op",
                     "pf_prox_step", "pf_admm_step"):
        assert required in names


def test_library_loads_and_exports_all_symbols():
    from paper_1904_10585_b200.build import build
    path = build()
    lib = ctypes.CDLL(path)
    for name in _declared():
        assert hasattr(lib, name), name


def test_argument_errors_are_synchronous_without_gpu():
    # pf_create validates shapes before touching the device
    from paper_1904_10585_b200 import load
    lib = load()
    h = ctypes.c_void_p()
    assert lib.pf_create(100, 24, 4, 0, ctypes.byref(h)) == 2      # p not supported -> DIM
    assert lib.pf_create(10, 16, 4, 0, ctypes.byref(h)) == 2       # n < p -> DIM
    assert lib.pf_create(100, 16, 0, 0, ctypes.byref(h)) == 1      # degree < 1 -> ARG
    assert lib.pf_create(100, 16, 4, 4, ctypes.byref(h)) == 7      # dtype -> UNSUPPORTED
    assert lib.pf_create(100, 24, 4, 3, ctypes.byref(h)) == 2      # PF_FP64_I8: fp64's p set
    assert lib.pf_create(100, 16, 4, 1, ctypes.byref(h)) == 7      # PF_FP32 reserved
    # PF_TF32 (config 5): p in {64, 128, 256, 512}
    assert lib.pf_create(1000, 16, 4, 2, ctypes.byref(h)) == 2
    assert lib.pf_create(1000, 96, 4, 2, ctypes.byref(h)) == 2
    assert lib.pf_create(300, 512, 4, 2, ctypes.byref(h)) == 2     # n < p
    nid = ctypes.create_string_buffer(128)
    # distributed TF32 needs n % (16 * world) == 0 (no K box straddles two ranks' slabs)
    assert lib.pf_create_dist(1000, 64, 4, 2, nid, 0, 1, ctypes.byref(h)) == 2
    assert lib.pf_set_tf32_passes(None, 3) == 1
    assert lib.pf_set_tf32_schedule(None, 1, 3) == 1
    assert lib.pf_set_i8_slices(None, 7) == 1
    assert lib.pf_invalidate(None) == 1
    assert lib.pf_matmul(None, None, 0, None, 0, None, 0, None) == 1
    assert lib.pf_status_string(3) == b"PF_ERR_INTERVAL"
    # round-2 entries: null contexts / invalid arguments fail before any device work
    loop = ctypes.c_void_p()
    assert lib.pf_loop_create(0, ctypes.byref(loop)) == 1            # world < 1
    assert lib.pf_loop_create(17, ctypes.byref(loop)) == 1           # world > 16
    assert lib.pf_create_loop(100, 16, 4, 0, None, 0, ctypes.byref(h)) == 1  # no hub
    assert lib.pf_loop_destroy(None) == 1
    d = ctypes.c_int32(0)
    assert lib.pf_schedule_degree(None, 1.0, 0, ctypes.byref(d)) == 1
    assert lib.pf_svt_kick(None, None, 0, 1.0, 1.0, 1.0, None, None) == 1
    assert lib.pf_svt_filter(None, None, None, None, None, None, None, None, 0, 1.0, 0.1,
                             None) == 1
    assert lib.pf_rebuild(None, None, 0, None, None, 0, None) == 1
    assert lib.pf_admm_step_f(None, None, 0, None, 1.0, None, 0, None, None, 0, None, None) == 1
    cnt = ctypes.c_int32(0)
    assert lib.pf_overlap_timeline(None, None, None, 0, ctypes.byref(cnt)) == 1
    assert lib.pf_set_z_upper(None, 1) == 1


def test_product_does_not_import_oracle():
    import subprocess, sys
    code = ("import sys; sys.path.insert(0, %r); import paper_1904_10585_b200, "
            "paper_1904_10585_b200.solver; assert 'oracle' not in sys.modules" % ROOT)
    subprocess.check_call([sys.executable, "-c", code])
    for f in os.listdir(os.path.join(ROOT, "paper_1904_10585_b200")):
        if f.endswith(".py"):
            src = open(os.path.join(ROOT, "paper_1904_10585_b200", f)).read()
            assert "import oracle" not in src and "from oracle" not in src, f
