"""CPU tier: the C-ABI library builds, loads and exports exactly what
include/fkc_sw.h declares, and the ctypes mirrors match the C struct layout."""

import ctypes
import os
import re
import subprocess
import tempfile

import pytest

from paper_1107_2157_b200 import _native as N

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "fkc_sw.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(fkc_\w+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    L = N.lib()
    names = declared_functions()
    assert set(names) == set(N.EXPORTS), (names, N.EXPORTS)
    for name in names:
        assert hasattr(L, name), name
    assert L.fkc_abi_version() == N.ABI_VERSION == 4


def test_usage_errors_without_gpu():
    L = N.lib()
    # null args -> usage error, message set, no device touched
    assert L.fkc_sw_step(None, None) == N.FKC_EUSAGE
    assert b"null" in L.fkc_last_error()
    a = N.StepArgs()
    a.grid = N.Grid(0, 4, 8, 0, 0)
    assert L.fkc_sw_step(ctypes.byref(a), None) == N.FKC_EUSAGE
    a.grid = N.Grid(8, 8, 12, 0, 0)
    a.H = a.U = a.V = a.oH = a.oU = a.oV = 1024
    assert L.fkc_sw_step(ctypes.byref(a), None) == N.FKC_EUSAGE   # aliasing
    halo = (ctypes.c_int32 * 4)(3, 3, 0, 0)
    assert L.fkc_region_cpy(0, 16, 5, 5, 5, halo, 32, 5, None) == N.FKC_EDOMAIN  # HaloTooLarge
    # per-call schedule (fkc_sw_tune): invalid values are usage errors before any device work
    a.grid = N.Grid(8, 8, 12, 0, 0)
    a.H, a.U, a.V, a.oH, a.oU, a.oV = 1024, 2048, 3072, 4096, 5120, 6144
    a.dx = a.dy = 1.0
    for bad in (dict(seg=-1), dict(tail_rows=-2), dict(tail_waves=65), dict(order=3), dict(parity=2),
                dict(warps=3), dict(no_pdl=2), dict(no_alternate=-1)):
        a.tune = N.Tune(**bad)
        assert L.fkc_sw_step(ctypes.byref(a), None) == N.FKC_EUSAGE, bad
        assert b"tune" in L.fkc_last_error()
    a.tune = N.Tune()
    # fused exchange: a peer line needs bc NONE on its side, and wait/signal come in pairs
    a.grid = N.Grid(8, 8, 12, 0, 0)
    a.H, a.U, a.V, a.oH, a.oU, a.oV = 1024, 2048, 3072, 4096, 5120, 6144
    a.dx = a.dy = 1.0
    a.peer[2].p[0] = a.peer[2].p[1] = a.peer[2].p[2] = 8192
    a.peer[2].stride = 1
    assert L.fkc_sw_step(ctypes.byref(a), None) == N.FKC_EUSAGE
    assert b"NONE" in L.fkc_last_error()
    a.bc[2] = N.BC_NONE
    a.peer[2].stride = 7
    assert L.fkc_sw_step(ctypes.byref(a), None) == N.FKC_EUSAGE
    assert b"stride" in L.fkc_last_error()
    a.peer[2].stride = 1
    a.sync.counter = 1 << 20
    a.sync.wait[0] = 1 << 21
    assert L.fkc_sw_step(ctypes.byref(a), None) == N.FKC_EUSAGE
    assert b"together" in L.fkc_last_error()
    # native time loop: argument checks before any device work
    assert L.fkc_sw_advance_n(None, None) == N.FKC_EUSAGE
    la = N.LoopArgs()
    la.steps = -1
    assert L.fkc_sw_advance_n(ctypes.byref(la), None) == N.FKC_EUSAGE
    la.steps = 3
    la.step.sync.counter = 1 << 20
    assert L.fkc_sw_advance_n(ctypes.byref(la), None) == N.FKC_EUSAGE
    assert b"per-step" in L.fkc_last_error()
    la.step.sync.counter = None
    la.dt_from_slots = 1
    assert L.fkc_sw_advance_n(ctypes.byref(la), None) == N.FKC_EUSAGE
    la.dt_from_slots = 0
    la.steps = 0
    assert L.fkc_sw_advance_n(ctypes.byref(la), None) == N.FKC_OK       # nothing to do


def test_struct_layout_matches_header():
    probe = r"""
    #include <stdio.h>
    #include <stddef.h>
    #include "fkc_sw.h"
    int main(void) {
      printf("%zu %zu %zu\n", sizeof(fkc_grid), sizeof(fkc_sw_reduce), sizeof(fkc_sw_step_args));
      printf("%zu %zu %zu %zu %zu %zu\n", offsetof(fkc_sw_step_args, H), offsetof(fkc_sw_step_args, dx),
             offsetof(fkc_sw_step_args, dt_bound), offsetof(fkc_sw_step_args, bc),
             offsetof(fkc_sw_step_args, variant), offsetof(fkc_sw_step_args, red));
      printf("%zu %zu %zu %zu %zu %zu\n", sizeof(fkc_peer_line), sizeof(fkc_sync),
             offsetof(fkc_sw_step_args, peer), offsetof(fkc_sw_step_args, sync),
             offsetof(fkc_sync, counter), offsetof(fkc_sync, epoch));
      printf("%zu %zu %zu %zu\n", sizeof(fkc_sw_tune), offsetof(fkc_sw_step_args, tune),
             offsetof(fkc_sw_tune, parity), offsetof(fkc_sw_tune, no_alternate));
      printf("%zu %zu %zu %zu %zu %zu\n", sizeof(fkc_sw_loop_args), offsetof(fkc_sw_loop_args, first_step),
             offsetof(fkc_sw_loop_args, slots), offsetof(fkc_sw_loop_args, want_cfl),
             offsetof(fkc_sw_loop_args, use_graph), offsetof(fkc_sw_loop_args, host_slots));
      return 0;
    }
    """
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "p.c")
        open(c, "w").write(probe)
        exe = os.path.join(d, "p")
        subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), c, "-o", exe], check=True)
        out = subprocess.run([exe], capture_output=True, text=True, check=True).stdout.split()
    got = list(map(int, out))
    S = N.StepArgs
    want = [ctypes.sizeof(N.Grid), ctypes.sizeof(N.Reduce), ctypes.sizeof(S),
            S.H.offset, S.dx.offset, S.dt_bound.offset, S.bc.offset, S.variant.offset, S.red.offset,
            ctypes.sizeof(N.PeerLine), ctypes.sizeof(N.Sync), S.peer.offset, S.sync.offset,
            N.Sync.counter.offset, N.Sync.epoch.offset,
            ctypes.sizeof(N.Tune), S.tune.offset, N.Tune.parity.offset, N.Tune.no_alternate.offset,
            ctypes.sizeof(N.LoopArgs), N.LoopArgs.first_step.offset, N.LoopArgs.slots.offset,
            N.LoopArgs.want_cfl.offset, N.LoopArgs.use_graph.offset, N.LoopArgs.host_slots.offset]
    assert got == want


def test_sm100a_sass_present():
    """The shipped .so carries sm_100a SASS (no PTX-JIT dependence)."""
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", N.LIB_PATH],
                         capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_integration_c_example_compiles_and_links():
    """The C snippet of INTEGRATION.md section 3 compiles against
    include/fkc_sw.h and links against the library; run without a GPU it
    reports the usage error for null pointers (no device touched)."""
    doc = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    sec = doc[doc.index("## 3. C / C++ callers"):]
    snippet = sec[sec.index("```c") + 4:sec.index("```", sec.index("```c") + 4)]
    main = r"""
    int main(void) {
        int rc = one_step(8, 8, 32, 0, 0, 0, 0, 0, 0, 0.1, 0);
        return rc == FKC_EUSAGE ? 0 : 1;
    }
    """
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "ex.c")
        open(c, "w").write(snippet + main)
        exe = os.path.join(d, "ex")
        libdir = os.path.dirname(N.LIB_PATH)
        subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), c, "-o", exe, "-L", libdir, "-lfkc_sw",
                        f"-Wl,-rpath,{libdir}"], check=True)
        r = subprocess.run([exe], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert "null" in r.stderr


C_MAIN = r"""
#include <stdlib.h>
#include <string.h>
#include <cuda_runtime.h>

/* reads nx ny K and the initial H,U,V ((ny+2) x (nx+2) f32 each) from argv[1];
 * writes the state after one_step (fast) and after many_steps (exact, K steps)
 * to argv[2] */
int main(int argc, char** argv) {
    FILE* f = fopen(argv[1], "rb");
    int hdr[3];
    if (!f || fread(hdr, 4, 3, f) != 3) return 10;
    const int nx = hdr[0], ny = hdr[1], K = hdr[2];
    const long W = nx + 2, Hh = ny + 2, pitch = (W + 31) / 32 * 32;
    const size_t n_host = (size_t)W * Hh;
    float* host = (float*)malloc(3 * n_host * 4);
    if (fread(host, 4, 3 * n_host, f) != 3 * n_host) return 11;
    fclose(f);
    void* base[6];
    float* ptr[6];
    for (int i = 0; i < 6; ++i) {
        /* the layout DeviceField uses: (ptr + 1 element) 128-B aligned, 31 readable floats before ptr */
        if (cudaMalloc(&base[i], (31 + Hh * pitch + 32) * 4) != cudaSuccess) return 12;
        ptr[i] = (float*)base[i] + 31;
    }
    for (int i = 0; i < 3; ++i)
        cudaMemcpy2D(ptr[i], pitch * 4, host + i * n_host, W * 4, W * 4, Hh, cudaMemcpyHostToDevice);
    FILE* o = fopen(argv[2], "wb");
    if (one_step(nx, ny, pitch, ptr[0], ptr[1], ptr[2], ptr[3], ptr[4], ptr[5], 0.05, 0) != FKC_OK) return 13;
    cudaDeviceSynchronize();
    for (int i = 3; i < 6; ++i) {
        cudaMemcpy2D(host, W * 4, ptr[i], pitch * 4, W * 4, Hh, cudaMemcpyDeviceToHost);
        fwrite(host, 4, n_host, o);
    }
    fkc_sw_step_args t = {0};
    t.grid = (fkc_grid){nx, ny, pitch, FKC_F32, 0};
    t.H = ptr[0]; t.U = ptr[1]; t.V = ptr[2]; t.oH = ptr[3]; t.oU = ptr[4]; t.oV = ptr[5];
    t.dx = t.dy = 1.0; t.dt = 0.05; t.g = 9.8;
    t.mode = FKC_MODE_EXACT;
    if (many_steps(&t, K, 0) != FKC_OK) { fprintf(stderr, "%s\n", fkc_last_error()); return 14; }
    if (cudaDeviceSynchronize() != cudaSuccess) return 15;
    for (int i = 0; i < 3; ++i) {
        cudaMemcpy2D(host, W * 4, ptr[(K % 2) ? 3 + i : i], pitch * 4, W * 4, Hh, cudaMemcpyDeviceToHost);
        fwrite(host, 4, n_host, o);
    }
    /* the host-state run: pinned initial state in, K exact steps, pinned state out */
    f = fopen(argv[1], "rb");
    if (!f || fread(hdr, 4, 3, f) != 3) return 17;
    float *hin[3], *hout[3];
    for (int i = 0; i < 3; ++i) {
        if (cudaMallocHost((void**)&hin[i], n_host * 4) != cudaSuccess) return 18;
        if (cudaMallocHost((void**)&hout[i], n_host * 4) != cudaSuccess) return 18;
        if (fread(hin[i], 4, n_host, f) != n_host) return 19;
    }
    fclose(f);
    if (run_from_host(&t, K, (const float* const*)hin, hout, W * 4, 0) != FKC_OK) {
        fprintf(stderr, "%s\n", fkc_last_error());
        return 20;
    }
    if (cudaDeviceSynchronize() != cudaSuccess) return 21;
    for (int i = 0; i < 3; ++i) fwrite(hout[i], 4, n_host, o);
    fclose(o);
    return 0;
}
"""


@pytest.mark.gpu
@pytest.mark.parametrize("nx,ny,K", [(1024, 700, 5), (516, 130, 4)])
def test_integration_c_example_on_device(nx, ny, K, tmp_path):
    """The INTEGRATION.md section 3 C example driven from a pure-C program
    on device memory it allocates itself (cudaMalloc, the padded layout):
    one_step (fast mode) within the fast tolerance of the oracle, the native
    time loop many_steps (exact mode, K steps) and the streamed host run
    run_from_host (pinned host state in and out) bit-identical to it."""
    import numpy as np
    from oracle import c_oracle
    from oracle import sw_oracle as so
    doc = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    sec = doc[doc.index("## 3. C / C++ callers"):]
    snippet = sec[sec.index("```c") + 4:sec.index("```", sec.index("```c") + 4)]
    c = tmp_path / "ex.c"
    c.write_text(snippet + C_MAIN)
    exe = tmp_path / "ex"
    libdir = os.path.dirname(N.LIB_PATH)
    cuda = "/usr/local/cuda"
    subprocess.run(["gcc", "-O1", "-I", os.path.join(ROOT, "include"), "-I", f"{cuda}/include", str(c), "-o", str(exe),
                    "-L", libdir, "-lfkc_sw", f"-Wl,-rpath,{libdir}", "-L", f"{cuda}/lib64", "-lcudart",
                    f"-Wl,-rpath,{cuda}/lib64"], check=True)
    H, U, V = so.random_state(nx, ny, "f32", seed=nx)
    inp = tmp_path / "in.bin"
    with open(inp, "wb") as f:
        f.write(np.array([nx, ny, K], np.int32).tobytes())
        for a in (H, U, V):
            f.write(np.ascontiguousarray(a, np.float32).tobytes())
    out = tmp_path / "out.bin"
    r = subprocess.run([str(exe), str(inp), str(out)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, (r.returncode, r.stderr)
    got = np.fromfile(out, np.float32).reshape(9, ny + 2, nx + 2)
    one = so.step(H, U, V, 1.0, 1.0, 0.05)
    for g, w in zip(got[:3], one):
        assert np.max(np.abs(g.astype(np.float64) - w)) <= 2e-5 * np.max(np.abs(w))
    want = c_oracle.run_fixed(H, U, V, K, 1.0, 1.0, 0.05)
    for g, w in zip(got[3:6], want):
        assert np.array_equal(g, w)
    for g, w in zip(got[6:], want):          # run_from_host: the streamed host run, same bits
        assert np.array_equal(g, w)


def test_integration_python_binding_matches_header():
    """INTEGRATION.md section 2 (the ctypes binding a maintainer of fkc would
    add) executes against the built library, and every structure it declares
    has the size and field offsets of the repo's own mirrors (which
    test_struct_layout_matches_c checks against the C header)."""
    md = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    sec = md[md.index("## 2. The binding"):md.index("## 3.")]
    code = re.search(r"```python\n(.*?)```", sec, flags=re.S).group(1)
    ns = {}
    old = os.environ.get("FKC_LIB")
    os.environ["FKC_LIB"] = N.LIB_PATH
    try:
        exec(compile(code, "INTEGRATION.md", "exec"), ns)   # noqa: S102 -- the documented binding itself
    finally:
        if old is None:
            os.environ.pop("FKC_LIB", None)
        else:
            os.environ["FKC_LIB"] = old
    for name in ("Grid", "Reduce", "PeerLine", "Sync", "Tune", "StepArgs", "LoopArgs"):
        mine, doc = getattr(N, name), ns[name]
        assert ctypes.sizeof(doc) == ctypes.sizeof(mine), name
        assert [f[0] for f in doc._fields_] == [f[0] for f in mine._fields_], name
        for f in mine._fields_:
            assert getattr(doc, f[0]).offset == getattr(mine, f[0]).offset, (name, f[0])
    assert callable(ns["advance"]) and callable(ns["run_host"])


def test_round2_usage_errors_without_gpu():
    """ABI 4 additions reject bad arguments before any device work: the CFL
    board fields of fkc_sync, the PDL flag, and fkc_sw_run_host's argument
    checks (CFL dt, periodic rows, host pitch, null pointers)."""
    L = N.lib()
    a = N.StepArgs()
    a.grid = N.Grid(8, 8, 12, 0, 0)
    a.H, a.U, a.V, a.oH, a.oU, a.oV = 1024, 2048, 3072, 4096, 5120, 6144
    a.dx = a.dy = 1.0
    a.sync.flags = 2                                    # unknown flag bit
    assert L.fkc_sw_step(ctypes.byref(a), None) == N.FKC_EUSAGE
    assert b"flags" in L.fkc_last_error()
    a.sync.flags = 0
    a.sync.cfl_board = 8192
    a.sync.cfl_nranks, a.sync.cfl_rank = 9, 0            # more ranks than the board holds
    assert L.fkc_sw_step(ctypes.byref(a), None) == N.FKC_EUSAGE
    a.sync.cfl_nranks, a.sync.cfl_rank = 2, 2            # rank out of range
    assert L.fkc_sw_step(ctypes.byref(a), None) == N.FKC_EUSAGE
    a.sync.cfl_rank = 1                                  # counter / peer boards missing
    assert L.fkc_sw_step(ctypes.byref(a), None) == N.FKC_EUSAGE
    a.sync.cfl_counter = 12288
    assert L.fkc_sw_step(ctypes.byref(a), None) == N.FKC_EUSAGE
    assert b"cfl_peers" in L.fkc_last_error()
    # fkc_sw_run_host
    lp = N.LoopArgs()
    lp.step = N.StepArgs()
    lp.step.grid = N.Grid(8, 8, 12, 0, 0)
    lp.step.H, lp.step.U, lp.step.V, lp.step.oH, lp.step.oU, lp.step.oV = 1024, 2048, 3072, 4096, 5120, 6144
    lp.step.dx = lp.step.dy = 1.0
    lp.steps = 2
    vp3 = ctypes.c_void_p * 3
    src, dst = vp3(64, 128, 192), vp3(256, 320, 384)
    assert L.fkc_sw_run_host(None, src, dst, 40, 0, None) == N.FKC_EUSAGE
    assert L.fkc_sw_run_host(ctypes.byref(lp), src, vp3(256, 0, 384), 40, 0, None) == N.FKC_EUSAGE
    assert L.fkc_sw_run_host(ctypes.byref(lp), src, dst, 8, 0, None) == N.FKC_EUSAGE        # pitch < row
    assert b"pitch" in L.fkc_last_error()
    lp.dt_from_slots = 1
    lp.slots = 4096
    assert L.fkc_sw_run_host(ctypes.byref(lp), src, dst, 40, 0, None) == N.FKC_EUSAGE
    assert b"fixed dt" in L.fkc_last_error()
    lp.dt_from_slots = 0
    lp.step.bc = N.bc_array((N.BC_REFLECTIVE, N.BC_REFLECTIVE, N.BC_PERIODIC, N.BC_PERIODIC))
    assert L.fkc_sw_run_host(ctypes.byref(lp), src, dst, 40, 0, None) == N.FKC_EUSAGE
    assert b"periodic" in L.fkc_last_error()


def test_streamable_rules():
    """swdemo.run's choice of the streamed host path (host state + host
    output + fixed dt + non-periodic rows + the TMA layout + >= 2^20 cells,
    contiguous host arrays of one pitch) -- host logic, no device."""
    import numpy as np

    from paper_1107_2157_b200 import swdemo
    from paper_1107_2157_b200.field import Field

    def st(nx, ny, order="C"):
        return swdemo.SWState(*(Field.from_array(np.ones((ny + 2, nx + 2), np.float32, order=order), "f32")
                                for _ in range(3)))
    big = st(1024, 1024)
    cfg = swdemo.SWConfig(nx=1024, ny=1024, steps=3, dt=0.05)
    assert swdemo._streamable(cfg, big, None)
    assert swdemo._streamable(cfg, big, st(1024, 1024))
    assert not swdemo._streamable(swdemo.SWConfig(nx=1024, ny=1024, steps=3), big, None)          # CFL dt
    assert not swdemo._streamable(swdemo.SWConfig(nx=1024, ny=1024, steps=3, dt=0.05, boundary="periodic"),
                                  big, None)
    assert not swdemo._streamable(swdemo.SWConfig(nx=1024, ny=1024, steps=3, dt=0.05, variant="generic"),
                                  big, None)
    assert not swdemo._streamable(cfg, st(1024, 1024, order="F"), None)                           # layout
    small = swdemo.SWConfig(nx=512, ny=512, steps=3, dt=0.05)
    assert not swdemo._streamable(small, st(512, 512), None)                                       # < 2^20 cells
    odd = swdemo.SWConfig(nx=1026, ny=1024, steps=3, dt=0.05)
    assert not swdemo._streamable(odd, st(1026, 1024), None)                                       # nx % 4
