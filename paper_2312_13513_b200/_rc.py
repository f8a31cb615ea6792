"""ctypes binding of include/rc.h (argument marshalling only).

Every computation of the path runs in librc_b200.so's sm_100a kernels; this
module only builds the C structs from numpy/torch objects and checks return
codes.  There is no CPU fallback: if the library is missing, importing
`lib()` raises.
"""
import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.environ.get("RC_LIB") or os.path.join(HERE, "librc_b200.so")  # RC_LIB: A/B experiments (tools/ab.sh)

RC_OK, RC_EINVAL, RC_ENOMEM, RC_ECUDA, RC_EALIGN, RC_EUNSUPPORTED, RC_EDTMISMATCH = 0, -1, -2, -3, -4, -5, -6
RC_MODE_H, RC_MODE_T = 0, 1
RC_BF16, RC_TF32, RC_TF32X3 = 0, 1, 2
RC_MLP_LAYERWISE, RC_MLP_SHARED, RC_MLP_SERIAL = 1, 2, 4
DIAG_NAMES = ["newton_bisect", "newton_maxit", "nonfinite", "negY_in", "negY_out"]


class RcError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"rc error {code}: {msg}")
        self.code = code


class rc_mech_desc(C.Structure):
    _fields_ = [("ns", C.c_int32), ("ne", C.c_int32), ("W_elem", C.c_void_p), ("atoms", C.c_void_p),
                ("nasa_lo", C.c_void_p), ("nasa_hi", C.c_void_p), ("T_lo", C.c_void_p), ("T_mid", C.c_void_p),
                ("T_hi", C.c_void_p), ("visc", C.c_void_p), ("cond", C.c_void_p), ("diff", C.c_void_p),
                ("inert", C.c_void_p)]


class rc_mlp_desc(C.Structure):
    _fields_ = [("n_nets", C.c_int32), ("hidden", C.c_int32 * 3), ("species_of_net", C.c_void_p),
                ("params", C.c_void_p), ("x_mean", C.c_void_p), ("x_std", C.c_void_p), ("y_mean", C.c_void_p),
                ("y_std", C.c_void_p), ("lambda_bc", C.c_double), ("dt", C.c_double), ("precision", C.c_int32),
                ("flags", C.c_int32)]


class rc_cells(C.Structure):
    _fields_ = [("n", C.c_int64), ("ld", C.c_int64), ("mode", C.c_int32), ("h", C.c_void_p), ("T", C.c_void_p),
                ("p", C.c_void_p), ("Y", C.c_void_p), ("cp", C.c_void_p), ("rho", C.c_void_p), ("mu", C.c_void_p),
                ("lam", C.c_void_p), ("D", C.c_void_p), ("wdot", C.c_void_p), ("qdot", C.c_void_p),
                ("o", C.c_void_p), ("dt", C.c_double), ("red", C.c_void_p), ("diag", C.c_void_p),
                ("tau_mix", C.c_void_p)]


class rc_kin_desc(C.Structure):
    _fields_ = [("nr", C.c_int32), ("nu_f", C.c_void_p), ("nu_r", C.c_void_p), ("type", C.c_void_p),
                ("reversible", C.c_void_p), ("A", C.c_void_p), ("b", C.c_void_p), ("Ea", C.c_void_p),
                ("eff", C.c_void_p), ("A0", C.c_void_p), ("b0", C.c_void_p), ("Ea0", C.c_void_p), ("troe", C.c_void_p)]


EXPORTS = {
    # name: (restype, argtypes)
    "rc_mech_create": (C.c_int, [C.POINTER(rc_mech_desc), C.POINTER(C.c_void_p)]),
    "rc_mech_destroy": (None, [C.c_void_p]),
    "rc_mech_ns": (C.c_int, [C.c_void_p]),
    "rc_mlp_create": (C.c_int, [C.c_void_p, C.POINTER(rc_mlp_desc), C.POINTER(C.c_void_p)]),
    "rc_mlp_destroy": (None, [C.c_void_p]),
    "rc_workspace_bytes": (C.c_size_t, [C.c_void_p, C.c_void_p, C.c_int64]),
    "rc_thermo": (C.c_int, [C.c_void_p, C.POINTER(rc_cells), C.c_void_p]),
    "rc_transport": (C.c_int, [C.c_void_p, C.POINTER(rc_cells), C.c_void_p]),
    "rc_chem": (C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(rc_cells), C.c_void_p, C.c_size_t, C.c_void_p]),
    "rc_step": (C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(rc_cells), C.c_void_p, C.c_size_t, C.c_void_p]),
    "rc_partition": (C.c_int, [C.c_int64, C.c_int, C.c_int, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "rc_combine_reductions": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]),
    "rc_kin_create": (C.c_int, [C.c_void_p, C.POINTER(rc_kin_desc), C.POINTER(C.c_void_p)]),
    "rc_kin_destroy": (None, [C.c_void_p]),
    "rc_kinetics": (C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(rc_cells), C.c_void_p]),
    "rc_laplacian": (C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(rc_cells), C.c_void_p, C.c_void_p, C.c_void_p,
                               C.c_void_p, C.c_int, C.c_void_p]),
    "rc_ldu_to_csr": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                C.c_void_p]),
    "rc_pack_planes": (C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(rc_cells), C.c_void_p, C.c_void_p, C.c_void_p]),
    "rc_last_launch_count": (C.c_int64, []),
    "rc_profile_enable": (C.c_int, [C.c_int]),
    "rc_profile_read": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int]),
    "rc_overlap_read": (C.c_int, [C.c_void_p, C.c_int]),
    "rc_profile_timeline": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int]),
    "rc_last_error": (C.c_char_p, []),
    "rc_version": (C.c_char_p, []),
}

_lib = None


def lib():
    """Load librc_b200.so (raises if it was not built: there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(SO):
            raise ImportError(f"{SO} not built; run `python -m paper_2312_13513_b200.build` (no CPU fallback exists)")
        L = C.CDLL(SO)
        for name, (res, args) in EXPORTS.items():
            if os.environ.get("RC_LIB") and not hasattr(L, name):
                continue  # an older build under A/B comparison (tools/ab.sh) may lack newer entry points
            f = getattr(L, name)
            f.restype, f.argtypes = res, args
        _lib = L
    return _lib


def check(code):
    if code != RC_OK:
        raise RcError(code, lib().rc_last_error().decode())
    return code


def _np(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


def _ptr(t):
    """device/host pointer of a torch tensor or numpy array (None -> NULL)."""
    if t is None:
        return None
    if hasattr(t, "data_ptr"):
        return t.data_ptr()
    return t.ctypes.data


def rc_partition(n_global, rank, world):
    b, e = C.c_int64(), C.c_int64()
    check(lib().rc_partition(n_global, rank, world, C.byref(b), C.byref(e)))
    return b.value, e.value


class Mechanism:
    """rc_mech handle built from a mechanism-table dict (keys of workload.load_mech)."""

    def __init__(self, m: dict):
        keep = {k: _np(m[k], dt) for k, dt in [
            ("W_elem", np.float64), ("atoms", np.int32), ("nasa_lo", np.float64), ("nasa_hi", np.float64),
            ("T_lo", np.float64), ("T_mid", np.float64), ("T_hi", np.float64), ("visc", np.float64),
            ("cond", np.float64), ("diff", np.float64), ("inert", np.uint8)]}
        d = rc_mech_desc(int(m["ns"]), int(m["ne"]), *[keep[k].ctypes.data for k in [
            "W_elem", "atoms", "nasa_lo", "nasa_hi", "T_lo", "T_mid", "T_hi", "visc", "cond", "diff", "inert"]])
        h = C.c_void_p()
        check(lib().rc_mech_create(C.byref(d), C.byref(h)))
        self.h = h
        self.ns = int(m["ns"])

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.rc_mech_destroy(self.h)
            self.h = None


class MLPBundle:
    """rc_mlp handle from a bundle dict (keys of workload.make_bundle)."""

    def __init__(self, mech: Mechanism, b: dict, precision: int = RC_BF16, flags: int = 0):
        self.keep = {k: _np(b[k], np.float64) for k in ["params", "x_mean", "x_std", "y_mean", "y_std"]}
        self.keep["species_of_net"] = _np(b["species_of_net"], np.int32)
        d = rc_mlp_desc(int(b["n_nets"]), (C.c_int32 * 3)(*b["hidden"]), self.keep["species_of_net"].ctypes.data,
                        self.keep["params"].ctypes.data, self.keep["x_mean"].ctypes.data,
                        self.keep["x_std"].ctypes.data, self.keep["y_mean"].ctypes.data,
                        self.keep["y_std"].ctypes.data, float(b["lambda_bc"]), float(b["dt"]), int(precision), int(flags))
        if b.get("shared"):
            d.flags |= RC_MLP_SHARED  # one shared net with n_nets outputs (NEXT-2)
        h = C.c_void_p()
        check(lib().rc_mlp_create(mech.h, C.byref(d), C.byref(h)))
        self.h = h
        self.n_nets = int(b["n_nets"])
        self.dt = float(b["dt"])
        self.mech = mech
        del self.keep  # host copies are not needed after create (the library copied them)

    def workspace_bytes(self, n):
        return int(lib().rc_workspace_bytes(self.mech.h, self.h, int(n)))

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.rc_mlp_destroy(self.h)
            self.h = None


class Kinetics:
    """rc_kin handle (detailed kinetics, NEXT-3) from a workload.load_kinetics() dict (SI)."""

    KEYS = [("nu_f", np.int32), ("nu_r", np.int32), ("type", np.int32), ("reversible", np.int32),
            ("A", np.float64), ("b", np.float64), ("Ea", np.float64), ("eff", np.float64), ("A0", np.float64),
            ("b0", np.float64), ("Ea0", np.float64), ("troe", np.float64)]

    def __init__(self, mech: Mechanism, k: dict):
        keep = {key: _np(k[key], dt) for key, dt in self.KEYS}
        d = rc_kin_desc(int(k["nr"]), *[keep[key].ctypes.data for key, _ in self.KEYS])
        h = C.c_void_p()
        check(lib().rc_kin_create(mech.h, C.byref(d), C.byref(h)))
        self.h = h
        self.nr = int(k["nr"])

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.rc_kin_destroy(self.h)
            self.h = None


def rc_kinetics(mech, kin, cells, stream=None):
    return check(lib().rc_kinetics(mech.h, kin.h, C.byref(cells), _stream(stream)))


class rc_mesh(C.Structure):
    _fields_ = [("nx", C.c_int32), ("ny", C.c_int32), ("nz", C.c_int32), ("dx", C.c_double), ("dy", C.c_double),
                ("dz", C.c_double)]


RC_LAP_GATHER, RC_LAP_ATOMIC = 0, 1


def rc_laplacian(mech, mesh, cells, upper, diag, halo_lo=None, halo_hi=None, mode=RC_LAP_GATHER, stream=None):
    """mesh = (nx, ny, nz, dx, dy, dz); upper [ns+1][3n], diag [ns+1][n] device tensors (NEXT-1)."""
    m = rc_mesh(*mesh)
    return check(lib().rc_laplacian(mech.h, C.byref(m), C.byref(cells), _ptr(halo_lo), _ptr(halo_hi), _ptr(upper),
                                    _ptr(diag), int(mode), _stream(stream)))


def rc_ldu_to_csr(mesh, nsys, upper, diag, row_ptr, col, val, stream=None):
    m = rc_mesh(*mesh)
    return check(lib().rc_ldu_to_csr(C.byref(m), int(nsys), _ptr(upper), _ptr(diag), _ptr(row_ptr), _ptr(col),
                                     _ptr(val), _stream(stream)))


def rc_pack_planes(mech, mesh, cells, bottom, top, stream=None):
    m = rc_mesh(*mesh)
    return check(lib().rc_pack_planes(mech.h, C.byref(m), C.byref(cells), _ptr(bottom), _ptr(top), _stream(stream)))


def make_cells(n, ld, mode, T, p, Y, h=None, cp=None, rho=None, mu=None, lam=None, D=None, wdot=None, qdot=None,
               o=None, dt=0.0, red=None, diag=None, tau_mix=None):
    """rc_cells struct from torch device tensors (component-major, stride ld)."""
    return rc_cells(int(n), int(ld), int(mode), _ptr(h), _ptr(T), _ptr(p), _ptr(Y), _ptr(cp), _ptr(rho), _ptr(mu),
                    _ptr(lam), _ptr(D), _ptr(wdot), _ptr(qdot), _ptr(o), float(dt), _ptr(red), _ptr(diag),
                    _ptr(tau_mix))


def _stream(stream):
    if stream is None:
        import torch
        return C.c_void_p(torch.cuda.current_stream().cuda_stream)
    return C.c_void_p(stream if isinstance(stream, int) else stream.cuda_stream)


def rc_thermo(mech, cells, stream=None):
    return check(lib().rc_thermo(mech.h, C.byref(cells), _stream(stream)))


def rc_transport(mech, cells, stream=None):
    return check(lib().rc_transport(mech.h, C.byref(cells), _stream(stream)))


def rc_chem(mech, mlp, cells, ws, stream=None):
    return check(lib().rc_chem(mech.h, mlp.h, C.byref(cells), _ptr(ws), ws.numel() * ws.element_size(),
                               _stream(stream)))


def rc_step(mech, mlp, cells, ws, stream=None):
    return check(lib().rc_step(mech.h, mlp.h if mlp is not None else None, C.byref(cells),
                               _ptr(ws) if ws is not None else None,
                               (ws.numel() * ws.element_size()) if ws is not None else 0, _stream(stream)))


def rc_combine_reductions(red_parts, diag_parts, red, diag, stream=None):
    """a6 over k sub-batches: red_parts [k][2] fp64, diag_parts [k][5] int64 (device tensors)."""
    return check(lib().rc_combine_reductions(_ptr(red_parts), _ptr(diag_parts), int(red_parts.shape[0]), _ptr(red),
                                             _ptr(diag), _stream(stream)))


def rc_last_launch_count():
    return int(lib().rc_last_launch_count())


STAGES = ["thermo", "transport", "prologue", "L1", "L2", "L3", "epilogue", "finalize", "L12", "L4", "kinetics",
          "laplacian", "csr", "L3_fill"]


def rc_profile_enable(on=True):
    return check(lib().rc_profile_enable(1 if on else 0))


def rc_profile_read(reset=True):
    """{stage: (total_ms, launches)} since the last reset (waits for the events)."""
    ms = np.zeros(len(STAGES), dtype=np.float64)
    cnt = np.zeros(len(STAGES), dtype=np.int64)
    check(lib().rc_profile_read(ms.ctypes.data, cnt.ctypes.data, 1 if reset else 0))
    return {s: (float(ms[i]), int(cnt[i])) for i, s in enumerate(STAGES)}


def rc_overlap_read(reset=True):
    """Layer-3 overlap counters since the last reset: {tiles_fill, pairs_gave_up, pairs_ran}."""
    out = np.zeros(3, dtype=np.int64)
    check(lib().rc_overlap_read(out.ctypes.data, 1 if reset else 0))
    return {"tiles_fill": int(out[0]), "pairs_gave_up": int(out[1]), "pairs_ran": int(out[2])}


def rc_profile_timeline(max_entries=100000):
    """[(stage name, start_ms, end_ms)] of the recorded launches (before rc_profile_read resets them)."""
    st = np.zeros(max_entries, dtype=np.int32)
    t0 = np.zeros(max_entries, dtype=np.float64)
    t1 = np.zeros(max_entries, dtype=np.float64)
    n = lib().rc_profile_timeline(st.ctypes.data, t0.ctypes.data, t1.ctypes.data, max_entries)
    if n < 0:
        check(n)
    n = min(n, max_entries)
    return [(STAGES[s] if 0 <= s < len(STAGES) else str(s), float(a), float(b)) for s, a, b in zip(st[:n], t0[:n], t1[:n])]
