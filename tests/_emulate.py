"""Rounding emulation of the MLP precision modes (test infrastructure).

An MLP that only rounds its operands -- bf16-RNE or tf32-RNE weights and activations,
fp32 accumulation, one rounding per activation, exact-erf GELU in fp32 -- run in torch on
the CPU.  Its error against the fp64 oracle is the floor any bf16 / TF32 tensor-core MLP
makes on the same cells; the GPU parity tests hold the kernels to a small multiple of it
(R17/R18) and tools/emulate_mlp.py prints it per net.  The o -> wdot map restates
SURVEY §8(c) steps 8-10 and is checked against the oracle's own wdot before use
(check_wdot_map).  Imports oracle/ (allowed: tests/ infrastructure), never the CUDA path.
"""
import numpy as np
import torch

import oracle
from workload.bundle import split_params


def rne_bf16(x):
    return x.to(torch.bfloat16).to(torch.float32)


def rne_tf32(x):
    # round-to-nearest-even to 10 explicit mantissa bits (tf32), kept in fp32
    i = x.contiguous().view(torch.int32).to(torch.int64)
    lsb = (i >> 13) & 1
    i = (i + 0xFFF + lsb) & ~0x1FFF
    return i.to(torch.int32).view(torch.float32)


def gelu_erf(x):
    return 0.5 * x * (1.0 + torch.erf(x * 0.7071067811865476))


def gelu_tanh(x):
    return 0.5 * x * (1.0 + torch.tanh(x * (0.7978845608 + 0.0356774081 * x * x)))


def gelu_bf16_ops(x):
    """tanh-form GELU with every operation rounded to bf16 (the round-1 bf16x2 code)."""
    r = rne_bf16
    c0, c1 = r(torch.tensor(0.7978846)), r(torch.tensor(0.0356774))
    xx = r(x * x)
    t = r(xx * c1 + c0)
    u = r(t * x)
    th = r(torch.tanh(u))
    hx = r(x * 0.5)
    return r(hx * th + hx)


def emulate_o(b, z64, variant):
    """o[net][cell] of the emulated MLP; z64 [n][d_in] fp64 from the oracle's prologue."""
    rnd = rne_tf32 if variant == "tf32" else rne_bf16
    outs = []
    z = rnd(torch.from_numpy(z64).to(torch.float32))
    for net in range(b["n_nets"]):
        W1, b1, W2, b2, W3, b3, W4, b4 = [torch.from_numpy(np.array(a)) for a in split_params(b, net)]
        h = z
        for l, (W, bb) in enumerate(((W1, b1), (W2, b2), (W3, b3))):
            acc = h @ rnd(W.to(torch.float32)).T + bb.to(torch.float32)
            if variant == "bf16_r01":
                a = gelu_bf16_ops(rne_bf16(acc)) if l < 2 else gelu_tanh(acc)
            elif variant == "bf16_tanh32":
                a = gelu_tanh(acc)
            else:
                a = gelu_erf(acc)
            h = a if (l == 2 and variant != "tf32") else rnd(a)
        o = h @ W4.to(torch.float32).T + b4.to(torch.float32)
        outs.append(o[:, 0].double().numpy())
    return np.array(outs)


def wdot_from_o(mech, b, P, T, rho, Y, o):
    """SURVEY §8(c) steps 8-10 restated: Delta = o sigma_y + mu_y; a = Yh^lam + lam Delta;
    Y* = a^(1/lam) (0 if a <= 0); dY = Y* - Yh; dY <- P dY; wdot = rho dY/dt; qdot = -sum h_k wdot_k."""
    lam = b["lambda_bc"]
    Yh = np.maximum(Y, 0.0)
    dY = np.zeros_like(Y)
    for net, s in enumerate(b["species_of_net"]):
        a = Yh[s] ** lam + lam * (o[net] * b["y_std"][net] + b["y_mean"][net])
        dY[s] = np.where(a > 0, np.maximum(a, 0) ** (1 / lam), 0.0) - Yh[s]
    w = rho[None] * (P @ dY) / b["dt"]
    om = oracle.Mech(mech)
    hk = np.array([[om.h_k(k, t) for t in T] for k in range(mech["ns"])])
    return w, -(hk * w).sum(0)


def rel(g, o):
    return float(np.linalg.norm(g - o) / np.linalg.norm(o))


def oracle_z(om, ob, T, p, Y):
    """z [n][d_in] from the oracle's own prologue."""
    return np.array([ob.prologue(om, T[i], p[i], Y[:, i])[0] for i in range(len(T))])


def check_wdot_map(mech, b, P, r, Y):
    w, q = wdot_from_o(mech, b, P, r["T"], r["rho"], Y, r["o"])
    assert rel(w, r["wdot"]) < 1e-10 and rel(q, r["qdot"]) < 1e-10, "restated o->wdot map disagrees with the oracle"


def emulated_errors(mech, b, c, r, variant):
    """(o, wdot, qdot) relative Frobenius errors of the emulated MLP against the oracle result
    r (oracle.step on cells c: p, Y), and the emulated o itself."""
    om, ob = oracle.Mech(mech), oracle.Mlp(b)
    P = om.projection()
    check_wdot_map(mech, b, P, r, c["Y"])
    z = oracle_z(om, ob, r["T"], c["p"], c["Y"])
    o = emulate_o(b, z, variant)
    w, q = wdot_from_o(mech, b, P, r["T"], r["rho"], c["Y"], o)
    return rel(o, r["o"]), rel(w, r["wdot"]), rel(q, r["qdot"]), o
