"""Space-time quadrature on the GPU: RHS projection and error norms
(reference fem.py:267-297 and :358-418).

The reference takes numpy callables; a GPU kernel needs the field as code,
so these entry points take C expressions in x, y, t (`pi` = KH_PI, math
functions of CUDA's libdevice: sin, cos, exp, pow, ...). The kernels in
csrc/quadrature.cu are compiled for sm_100a by NVRTC with the expressions
substituted (one compile per distinct expression set, cached per process)
and launched through the CUDA driver API on torch's current stream. The
quadrature tables are the host code's own (fem.triangle_rule,
fem._time_panels), so results agree with `fem.project_rhs` /
`fem.error_norms` (and the reference) to rounding (tests/test_quadrature.py,
tests/test_gpu_quadrature.py).
"""

import ctypes
import math
import os

import numpy as np

from .errors import DeviceError, DimensionMismatch
from .fem import _time_panels, error_quadrature, gauss_rule_01, triangle_rule

_SRC = os.path.join(os.path.dirname(os.path.abspath(__file__)), "csrc", "quadrature.cu")
_CACHE = {}


def _subst(expr):
    import re

    return "(" + re.sub(r"\bpi\b", "KH_PI", expr) + ")"


def cubin(defines):
    """NVRTC-compile csrc/quadrature.cu for sm_100a with the expression
    macros `defines` (no GPU needed); returns the cubin bytes."""
    from cuda.bindings import nvrtc

    with open(_SRC) as fh:
        body = fh.read()
    head = "".join(f"#define {k} {v}\n" for k, v in defines.items())
    src = (head + body).encode()
    err, prog = nvrtc.nvrtcCreateProgram(src, b"quadrature.cu", 0, [], [])
    _check(err, "nvrtcCreateProgram")
    opts = [b"--gpu-architecture=sm_100a", b"-std=c++17", b"-lineinfo"]
    err, = nvrtc.nvrtcCompileProgram(prog, len(opts), opts)
    if err != nvrtc.nvrtcResult.NVRTC_SUCCESS:
        _, size = nvrtc.nvrtcGetProgramLogSize(prog)
        log = b" " * size
        nvrtc.nvrtcGetProgramLog(prog, log)
        raise DeviceError("NVRTC compile of the quadrature kernels failed:\n" + log.decode(errors="replace"))
    err, size = nvrtc.nvrtcGetCUBINSize(prog)
    _check(err, "nvrtcGetCUBINSize")
    out = b" " * size
    err, = nvrtc.nvrtcGetCUBIN(prog, out)
    _check(err, "nvrtcGetCUBIN")
    nvrtc.nvrtcDestroyProgram(prog)
    return out


def _compile(defines):
    """(module, {name: function}) for the expression macros (cached)."""
    from cuda.bindings import driver

    key = tuple(sorted(defines.items()))
    if key in _CACHE:
        return _CACHE[key]
    err, mod = driver.cuModuleLoadData(cubin(defines))
    _check(err, "cuModuleLoadData")
    funcs = {}
    for name in (b"project_rhs_kernel", b"error_norms_kernel"):
        err, fn = driver.cuModuleGetFunction(mod, name)
        _check(err, "cuModuleGetFunction")
        funcs[name.decode()] = fn
    _CACHE[key] = (mod, funcs)
    return _CACHE[key]


def rhs_defines(f_expr):
    return {"KH_F": _subst(f_expr), "KH_U": "0.0", "KH_UX": "0.0", "KH_UY": "0.0", "KH_UT": "0.0"}


def error_defines(u_expr, ux_expr, uy_expr, ut_expr):
    return {"KH_F": "0.0", "KH_U": _subst(u_expr), "KH_UX": _subst(ux_expr), "KH_UY": _subst(uy_expr),
            "KH_UT": _subst(ut_expr)}


def _check(err, what):
    code = int(getattr(err, "value", err))
    if code != 0:
        raise DeviceError(f"{what} failed ({err})")


def _launch(fn, grid, block, args):
    """args: list of ctypes scalars (pointers as c_uint64)."""
    import torch
    from cuda.bindings import driver

    ptrs = (ctypes.c_void_p * len(args))(*[ctypes.addressof(a) for a in args])
    stream = torch.cuda.current_stream().cuda_stream
    err, = driver.cuLaunchKernel(fn, grid, 1, 1, block, 1, 1, 0, stream, ctypes.addressof(ptrs), 0)
    _check(err, "cuLaunchKernel")


def _tables(mesh_x, mesh_t, pts, wts, tq, tw, device):
    import torch

    if len(wts) > 64:
        raise DimensionMismatch("at most 64 spatial quadrature points")
    dev = torch.device(device)
    t = lambda a, dt=torch.float64: torch.as_tensor(np.array(a), dtype=dt).to(dev)
    q0, w0 = _time_panels(0, tq, tw)
    q1, w1 = _time_panels(1, tq, tw)
    tabs = dict(verts=t(mesh_x.vertices), tris=t(mesh_x.triangles, torch.int64), nodes=t(mesh_t.nodes),
                pts=t(pts), wts=t(wts), tq0=t(q0), tw0=t(w0), tq1=t(q1), tw1=t(w1))
    return tabs, len(wts), len(q0), len(q1)


def _common_args(tabs, n_tri, n_cells, nq, n0, n1):
    P = lambda x: ctypes.c_uint64(x.data_ptr())
    return [P(tabs["verts"]), P(tabs["tris"]), ctypes.c_int64(n_tri), P(tabs["nodes"]), ctypes.c_int(n_cells),
            P(tabs["pts"]), P(tabs["wts"]), ctypes.c_int(nq), P(tabs["tq0"]), P(tabs["tw0"]), ctypes.c_int(n0),
            P(tabs["tq1"]), P(tabs["tw1"]), ctypes.c_int(n1)]


def project_rhs_gpu(mesh_x, mesh_t, f_expr, quad_order=6, device="cuda"):
    """Cell averages of f(x, y, t) (a C expression) over triangle x interval
    cells, shape (n_triangles, n_cells) -- `fem.project_rhs` / reference
    fem.py:267-297 on the GPU. Returns a host array."""
    import torch

    from . import _native

    _native.require_cuda()
    pts, wts = triangle_rule(quad_order)
    tq, tw = gauss_rule_01((quad_order + 4) // 2)
    tabs, nq, n0, n1 = _tables(mesh_x, mesh_t, pts, wts, tq, tw, device)   # (makes the context current)
    _, funcs = _compile(rhs_defines(f_expr))
    n_tri, n_cells = mesh_x.n_triangles, mesh_t.n_cells
    out = torch.empty((n_tri, n_cells), dtype=torch.float64, device=tabs["verts"].device)
    total = n_tri * n_cells
    grid = max(1, min((total + 255) // 256, 148 * 32))
    _launch(funcs["project_rhs_kernel"], grid, 256,
            _common_args(tabs, n_tri, n_cells, nq, n0, n1) + [ctypes.c_uint64(out.data_ptr())])
    return out.cpu().numpy()


def error_norms_gpu(coeffs, mesh_x, mesh_t, u_expr, ux_expr, uy_expr, ut_expr, quad_order=None, device="cuda"):
    """(L2, H1-seminorm) space-time errors of the P1 x P1 function `coeffs`
    (n_vertices x N_t, boundary values included) against the exact solution
    given as C expressions (u, u_x, u_y, u_t) -- `fem.error_norms` /
    reference fem.py:358-418 on the GPU."""
    import torch

    from . import _native

    _native.require_cuda()
    if coeffs.shape != (mesh_x.n_vertices, mesh_t.n_cells):
        raise DimensionMismatch(f"coeffs shape {coeffs.shape} does not match "
                                f"{(mesh_x.n_vertices, mesh_t.n_cells)}")
    (pts, wts), (tq, tw) = error_quadrature(quad_order)
    tabs, nq, n0, n1 = _tables(mesh_x, mesh_t, pts, wts, tq, tw, device)
    _, funcs = _compile(error_defines(u_expr, ux_expr, uy_expr, ut_expr))
    full = np.hstack([np.zeros((mesh_x.n_vertices, 1)), np.asarray(coeffs, dtype=np.float64)])
    dev = tabs["verts"].device
    c = torch.as_tensor(np.ascontiguousarray(full)).to(dev)
    n_tri = mesh_x.n_triangles
    part = torch.empty((n_tri, 2), dtype=torch.float64, device=dev)
    grid = max(1, min((n_tri + 127) // 128, 148 * 32))
    _launch(funcs["error_norms_kernel"], grid, 128,
            _common_args(tabs, n_tri, mesh_t.n_cells, nq, n0, n1)
            + [ctypes.c_uint64(c.data_ptr()), ctypes.c_uint64(part.data_ptr())])
    s = part.sum(dim=0).cpu().numpy()
    return math.sqrt(s[0]), math.sqrt(s[1])
