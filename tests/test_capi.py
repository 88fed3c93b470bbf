"""T9: the C ABI of include/pico.h.  CPU tests load the library and call only
host-side paths (no compute); GPU tests exercise status codes end to end."""
import ctypes

import numpy as np
import pytest

import paper_2402_15253_b200 as pico
from paper_2402_15253_b200 import _lib


@pytest.fixture(scope="module")
def lib():
    from paper_2402_15253_b200 import build
    build.build()
    return pico.load()


def test_exports_every_header_symbol(lib):
    names = pico.header_functions()
    assert "pico_coreness" in names and "pico_coreness_ex" in names and "pico_coreness_host" in names
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_status_strings_and_version(lib):
    for code, name in _lib.STATUS.items():
        assert lib.pico_status_string(code).decode() == name
    assert lib.pico_status_string(99).decode() == "PICO_UNKNOWN"
    assert lib.pico_version() >= 100


def test_workspace_bytes_monotone(lib):
    a = pico.workspace_bytes(1000, 5000, "histocore")
    b = pico.workspace_bytes(1000, 50000, "histocore")
    c = pico.workspace_bytes(1000, 5000, "peelone")
    assert 0 < a < b and c > 0
    # histogram = 2m int32 slots dominate HistoCore's workspace
    assert b - a >= 4 * 2 * 45000
    assert pico.workspace_bytes(0, 0, "histocore") == 256


def test_host_side_argument_errors(lib):
    """Rejected before any device work, so safe without a GPU."""
    rp = np.zeros(3, dtype=np.int64)
    ci = np.zeros(2, dtype=np.int32)
    core = np.zeros(2, dtype=np.int32)
    f = lib.pico_coreness_ex
    P = rp.ctypes.data
    assert f(P, ci.ctypes.data, -1, 0, 0, core.ctypes.data, None, 0, None, 0, None) == 1
    assert f(P, ci.ctypes.data, 2, -1, 0, core.ctypes.data, None, 0, None, 0, None) == 1
    assert f(P, ci.ctypes.data, 2, 1, 7, core.ctypes.data, None, 0, None, 0, None) == 1
    assert b"unknown algo" in lib.pico_last_error()
    assert f(None, ci.ctypes.data, 2, 1, 0, core.ctypes.data, None, 0, None, 0, None) == 1
    assert f(P, None, 2, 1, 0, core.ctypes.data, None, 0, None, 0, None) == 1
    assert f(P, ci.ctypes.data, 2, 1, 0, None, None, 0, None, 0, None) == 1
    assert f(P, ci.ctypes.data, 1 << 31, 1, 0, core.ctypes.data, None, 0, None, 0, None) == 2
    # n == 0 is a no-op returning PICO_OK
    assert f(P, ci.ctypes.data, 0, 0, 0, None, None, 0, None, 0, None) == 0
    assert lib.pico_coreness(P, ci.ctypes.data, 0, 0, 1, None, None) == 0
    # too-small caller workspace
    assert f(P, ci.ctypes.data, 2, 1, 0, core.ctypes.data, None, 0, 1024, 16, None) == 1
    assert b"workspace too small" in lib.pico_last_error()
    # host entry point shares the checks
    assert lib.pico_coreness_host(P, ci.ctypes.data, -5, 1, 0, core.ctypes.data, None, 0, None) == 1
    assert lib.pico_coreness_host(P, ci.ctypes.data, 0, 0, 0, None, None, 0, None) == 0


def test_stats_struct_layout(tmp_path):
    """The ctypes mirror of pico_stats_t matches the C header field by field
    (offsets and size from gcc on include/pico.h)."""
    import subprocess
    from paper_2402_15253_b200.build import INCLUDE
    fields = [f for f, _ in _lib.Stats._fields_]
    src = tmp_path / "layout.c"
    src.write_text("#include <stdio.h>\n#include <stddef.h>\n#include \"pico.h\"\nint main(void){\n"
                   + "".join(f'printf("%zu\\n", offsetof(pico_stats_t, {f}));\n' for f in fields)
                   + 'printf("%zu\\n", sizeof(pico_stats_t));return 0;}\n')
    exe = tmp_path / "layout"
    subprocess.check_call(["gcc", "-I" + INCLUDE, str(src), "-o", str(exe)])
    got = [int(x) for x in subprocess.check_output([str(exe)]).split()]
    want = [getattr(_lib.Stats, f).offset for f in fields] + [ctypes.sizeof(_lib.Stats)]
    assert got == want


def test_python_api_refuses_cpu_tensors(lib):
    import torch
    rp = torch.zeros(3, dtype=torch.int64)
    ci = torch.zeros(2, dtype=torch.int32)
    with pytest.raises(ValueError, match="CUDA"):
        pico.coreness(rp, ci)


# ---------------------------------------------------------------- GPU
def _dev():
    import torch
    return torch.device("cuda:0")


@pytest.mark.gpu
def test_validate_rejects_malformed():
    import torch
    dev = _dev()

    def run(rp, ci, n):
        return pico.coreness(torch.tensor(rp, dtype=torch.int64, device=dev),
                             torch.tensor(ci, dtype=torch.int32, device=dev), flags=pico.F_VALIDATE)

    # good: path 0-1-2
    assert run([0, 1, 3, 4], [1, 0, 2, 1], 3).cpu().tolist() == [1, 1, 1]
    cases = {
        "self-loop": ([0, 2, 3, 4], [0, 1, 0, 1], 3),  # bad: 0-0 loop (also asym counts)
        "duplicate": ([0, 2, 4], [1, 1, 0, 0], 2),
        "asymmetric": ([0, 1, 1, 2], [1, 0], 3),
        "range": ([0, 1, 2], [5, 0], 2),
        "rowptr": ([0, 3, 2], [1, 0], 2),
    }
    for name, (rp, ci, n) in cases.items():
        if len(ci) % 2:
            continue
        with pytest.raises(pico.PicoError) as ei:
            run(rp, ci, n)
        assert ei.value.status == 6, name


@pytest.mark.gpu
def test_inputs_untouched_and_workspace():
    import torch
    import synth
    dev = _dev()
    rp, ci = synth.CONFIGS["R12"].build(device=dev)
    rp0, ci0 = rp.clone(), ci.clone()
    for algo in ("histocore", "peelone"):
        need = pico.workspace_bytes(rp.numel() - 1, ci.numel() // 2, algo)
        ws = torch.empty(need, dtype=torch.uint8, device=dev)
        a = pico.coreness(rp, ci, algo=algo, workspace=ws)
        b = pico.coreness(rp, ci, algo=algo)
        assert torch.equal(a, b)
        small = torch.empty(need // 2, dtype=torch.uint8, device=dev)
        with pytest.raises(pico.PicoError) as ei:
            pico.coreness(rp, ci, algo=algo, workspace=small)
        assert ei.value.status == 1
    assert torch.equal(rp, rp0) and torch.equal(ci, ci0)


@pytest.mark.gpu
def test_edgeless_and_isolated():
    import torch
    dev = _dev()
    rp = torch.zeros(6, dtype=torch.int64, device=dev)
    ci = torch.zeros(0, dtype=torch.int32, device=dev)
    for algo in ("histocore", "peelone"):
        assert pico.coreness(rp, ci, algo=algo).cpu().tolist() == [0] * 5


@pytest.mark.gpu
def test_host_entry_point_matches_device():
    import synth
    import oracle
    rp, ci = synth.to_numpy(*synth.CONFIGS["R12"].build())
    ref = oracle.bz(rp, ci)
    for algo in ("histocore", "peelone"):
        st = pico.Stats()
        core = pico.coreness_host(rp, ci, algo=algo, stats=st)
        assert np.array_equal(core, ref)


@pytest.mark.gpu
def test_invalid_graph_terminates():
    """An input that breaks the CSR contract (asymmetric, duplicate arcs) is
    not validated by default, but the call must still return -- a status or
    some coreness -- instead of hanging the device."""
    import torch
    dev = torch.device("cuda:0")
    rng = np.random.default_rng(3)
    n = 2000
    deg = rng.integers(0, 40, n)
    rp = np.zeros(n + 1, dtype=np.int64)
    rp[1:] = np.cumsum(deg)
    ci = rng.integers(0, n, rp[-1]).astype(np.int32)  # random one-way arcs with repeats
    if ci.size % 2:
        ci = ci[:-1]
        rp[-1] -= 1
        rp = np.minimum(rp, ci.size)
    r = torch.from_numpy(rp).to(dev)
    c = torch.from_numpy(ci).to(dev)
    for algo in ("histocore", "peelone"):
        for fl in (0, pico.F_PULL_ALWAYS, pico.F_PUSH_ONLY):
            if algo == "peelone" and fl:
                continue
            try:
                pico.coreness(r, c, algo=algo, flags=fl)
                torch.cuda.synchronize()
            except pico.PicoError as e:
                assert e.status in (4, 6)
    with pytest.raises(pico.PicoError) as ei:
        pico.coreness(r, c, flags=pico.F_VALIDATE)
    assert ei.value.status == 6


def test_sharded_abi_argument_checks():
    """The NCCL sharded entry points reject bad arguments without a GPU."""
    lib = pico.load()
    uid = (ctypes.c_uint8 * 128)()
    h = ctypes.c_void_p()
    assert lib.pico_comm_init(0, 0, uid, ctypes.byref(h)) == 1       # nranks < 1
    assert lib.pico_comm_init(2, 2, uid, ctypes.byref(h)) == 1       # rank out of range
    assert lib.pico_comm_init(1, 0, uid, None) == 1                  # NULL out
    assert lib.pico_coreness_sharded(None, None, None, 4, 2, 0, 4, 0, None, None) == 1  # NULL comm
    assert lib.pico_comm_size(None, None, None) == 1
    assert lib.pico_comm_destroy(None) == 0


def test_clamp_hammer_argument_errors(lib):
    """Rejected before any device work."""
    fin, gt, k1 = ctypes.c_int32(), ctypes.c_int64(), ctypes.c_int64()
    args = (ctypes.byref(fin), ctypes.byref(gt), ctypes.byref(k1), None)
    assert lib.pico_clamp_hammer(3, 5, 1, 4, *args) == 1
    assert lib.pico_clamp_hammer(0, 5, 1, -1, *args) == 1
    assert lib.pico_clamp_hammer(0, 5, -1, 4, *args) == 1
    assert lib.pico_clamp_hammer(0, 5, 1, 4, None, ctypes.byref(gt), ctypes.byref(k1), None) == 1


@pytest.mark.gpu
@pytest.mark.parametrize("mode", [0, 1, 2])
@pytest.mark.parametrize("d,k,c", [(10, 3, 4), (10, 3, 7), (10, 3, 8), (10, 3, 100_000), (1000, 2, 997),
                                   (1 << 20, 7, 1 << 20), (5, 5, 64), (4, 6, 32), (9, 0, 1), (9, 8, 0)])
def test_clamp_law_hammer(mode, d, k, c):
    """SURVEY 4 T5 / S:137 / P:273: c concurrent atomicSub>=k calls on one cell
    holding d end at max(k, d - c); exactly min(c, d - k) of them observe an old
    value > k, and exactly one observes k + 1 (the same-level push) iff
    k < d <= k + c -- for every clamp implementation the PeelOne kernels use."""
    import torch
    torch.cuda.init()
    fin, gt, k1 = pico.clamp_hammer(mode, d, k, c)
    assert fin == max(k, d - c) if d > k else fin == d
    assert gt == min(c, max(d - k, 0))
    assert k1 == (1 if k < d <= k + c else 0)


@pytest.mark.gpu
@pytest.mark.parametrize("cfg", ["R12", "C1"])
@pytest.mark.parametrize("algo", [0, 1])
def test_north_star_seven_argument_call(lib, cfg, algo):
    """The literal north-star entry point pico_coreness(rowptr, colidx, n, m,
    algo, core_out, stream) on real graphs, called through the
    C ABI with raw device pointers: bit-exact against the BZ oracle."""
    import torch
    import oracle
    import synth
    dev = torch.device("cuda:0")
    rp, ci = synth.CONFIGS[cfg].build(device=dev)
    n, m = rp.numel() - 1, ci.numel() // 2
    out = torch.full((n,), -1, dtype=torch.int32, device=dev)
    s = torch.cuda.current_stream(dev)
    rc = lib.pico_coreness(rp.data_ptr(), ci.data_ptr(), n, m, algo, out.data_ptr(), ctypes.c_void_p(s.cuda_stream))
    assert rc == 0, lib.pico_last_error()
    ref = oracle.bz(*synth.to_numpy(rp, ci))
    assert np.array_equal(out.cpu().numpy(), ref)
