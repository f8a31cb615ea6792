"""B200-native (sm_100a) cell-local reactive update of arXiv 2312.13513.

Per finite-volume cell: enthalpy -> temperature Newton inversion on NASA-7
polynomials, cp / rho, Wilke-Mathur mixture transport and mixture-averaged
diffusivities, and the per-species GELU-MLP chemistry step with Box-Cox
transform and element-conserving projection (§2
§3.1).  The compute lives in librc_b200.so (C ABI: include/rc.h); this
package is the thin Python binding plus torch-backed device buffers.
PyTorch is used only for device memory, streams and torch.distributed.
"""
import numpy as np

from . import _rc
from ._rc import (RC_BF16, RC_TF32, RC_TF32X3, RC_MODE_H, RC_MODE_T, DIAG_NAMES, Kinetics, Mechanism, MLPBundle, RcError,
                  lib, make_cells, rc_chem, rc_kinetics, rc_laplacian, rc_ldu_to_csr, rc_pack_planes, RC_LAP_GATHER,
                  RC_LAP_ATOMIC, rc_combine_reductions, rc_last_launch_count, rc_partition, rc_profile_enable, rc_profile_read, rc_step,
                  rc_thermo, rc_transport, STAGES, RC_MLP_LAYERWISE, RC_MLP_SHARED, RC_MLP_SERIAL, rc_overlap_read,
                  rc_profile_timeline)

__all__ = ["Mechanism", "MLPBundle", "Kinetics", "rc_kinetics", "rc_laplacian", "rc_ldu_to_csr", "rc_pack_planes",
           "RC_LAP_GATHER", "RC_LAP_ATOMIC", "CellState", "RcError", "RC_BF16", "RC_TF32", "RC_TF32X3", "RC_MODE_H", "RC_MODE_T",
           "rc_step", "rc_thermo", "rc_transport", "rc_chem", "rc_partition", "rc_combine_reductions",
           "rc_last_launch_count", "lib",
           "DIAG_NAMES", "make_cells", "rc_profile_enable", "rc_profile_read", "STAGES", "aligned_workspace",
           "RC_MLP_LAYERWISE", "RC_MLP_SHARED", "RC_MLP_SERIAL", "rc_overlap_read", "rc_profile_timeline"]


class CellState:
    """Component-major device buffers for n cells (torch tensors, fp64; o fp32).

    Inputs: h, T, p, Y[ns][ld].  Outputs: cp, rho, mu, lam, D[ns][ld], wdot[ns][ld],
    qdot, o[n_nets][ld], red[2], diag[5].
    """

    def __init__(self, n, ns, n_nets=0, device="cuda", ld=None, outputs=("cp", "rho", "mu", "lam", "D", "wdot", "qdot", "o"),
                 sources=False):
        """sources=True allocates wdot / qdot without an MLP (detailed kinetics, rc_kinetics)."""
        import torch
        self.n, self.ns, self.n_nets = int(n), int(ns), int(n_nets)
        self.ld = int(ld) if ld is not None else max(2, (self.n + 31) // 32 * 32)
        f64 = dict(dtype=torch.float64, device=device)
        ld = self.ld
        self.h = torch.zeros(ld, **f64)
        self.T = torch.zeros(ld, **f64)
        self.p = torch.zeros(ld, **f64)
        self.Y = torch.zeros(ns, ld, **f64)
        self.cp = torch.zeros(ld, **f64) if "cp" in outputs else None
        self.rho = torch.zeros(ld, **f64)
        self.mu = torch.zeros(ld, **f64) if "mu" in outputs else None
        self.lam = torch.zeros(ld, **f64) if "lam" in outputs else None
        self.D = torch.zeros(ns, ld, **f64) if "D" in outputs else None
        self.wdot = torch.zeros(ns, ld, **f64) if ("wdot" in outputs and (n_nets or sources)) else None
        self.qdot = torch.zeros(ld, **f64) if ("qdot" in outputs and (n_nets or sources)) else None
        self.o = torch.zeros(max(n_nets, 1), ld, dtype=torch.float32, device=device) if ("o" in outputs and n_nets) else None
        self.red = torch.zeros(2, **f64)
        self.diag = torch.zeros(5, dtype=torch.int64, device=device)
        self.tau_mix = None  # LES PaSR mixing time [ld] (set_tau_mix); None = laminar

    def load(self, T, p, Y, h=None):
        """Copy host (numpy) inputs into the device buffers (first n columns)."""
        import torch
        n = self.n
        self.T[:n].copy_(torch.from_numpy(np.ascontiguousarray(T, dtype=np.float64)))
        self.p[:n].copy_(torch.from_numpy(np.ascontiguousarray(p, dtype=np.float64)))
        self.Y[:, :n].copy_(torch.from_numpy(np.ascontiguousarray(Y, dtype=np.float64)))
        if h is not None:
            self.h[:n].copy_(torch.from_numpy(np.ascontiguousarray(h, dtype=np.float64)))
        return self

    def set_tau_mix(self, tau):
        """LES PaSR subgrid mixing time per cell (host array, s); None switches PaSR off."""
        import torch
        if tau is None:
            self.tau_mix = None
            return self
        if self.tau_mix is None:
            self.tau_mix = torch.zeros(self.ld, dtype=torch.float64, device=self.T.device)
        self.tau_mix[:self.n].copy_(torch.from_numpy(np.ascontiguousarray(tau, dtype=np.float64)))
        return self

    def cells(self, mode=RC_MODE_H, dt=0.0, chem=True, transport=True):
        return make_cells(self.n, self.ld, mode, self.T, self.p, self.Y, h=self.h, cp=self.cp, rho=self.rho,
                          mu=self.mu if transport else None, lam=self.lam if transport else None,
                          D=self.D if transport else None, wdot=self.wdot if chem else None,
                          qdot=self.qdot if chem else None, o=self.o if chem else None, dt=dt, red=self.red,
                          diag=self.diag, tau_mix=self.tau_mix)

    def host(self):
        """dict of numpy copies of every buffer (first n columns)."""
        n = self.n
        out = {}
        for k in ("h", "T", "p", "cp", "rho", "mu", "lam", "qdot"):
            t = getattr(self, k)
            if t is not None:
                out[k] = t[:n].cpu().numpy()
        for k in ("Y", "D", "wdot", "o"):
            t = getattr(self, k)
            if t is not None:
                out[k] = t[:, :n].cpu().numpy()
        out["red"] = self.red.cpu().numpy()
        out["diag"] = self.diag.cpu().numpy()
        return out


def aligned_workspace(mlp, n, device="cuda"):
    """Caller-owned, 256-byte aligned workspace from torch's caching allocator (the
    stream-ordered-allocator role of PAPER.md:216)."""
    import torch
    nbytes = mlp.workspace_bytes(n)
    buf = torch.empty(nbytes + 256, dtype=torch.uint8, device=device)
    off = (-buf.data_ptr()) % 256
    return buf[off:off + nbytes]
