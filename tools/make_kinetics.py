"""Write data/mech/h2_9sp_kin.json: the 9-species / 12-reaction H2/air mechanism of the paper's
quasi-DNS runs ("9 species and 12 reactions") for the detailed-kinetics source term
(reading R21), converted once to SI (kmol, m^3, J/kmol).

The paper gives no rate constants.  The set below is the 12-step H2/air skeleton of the San Diego
lineage (Boivin, Jimenez, Sanchez & Williams, Proc. Combust. Inst. 33, 2011) with rate constants
recalled from the public literature in CGS units (cm, mol, s, kJ/mol); every reaction is taken
reversible (reverse rate from the equilibrium constant of the NASA tables), three-body and falloff
forms as listed.  GPU-vs-oracle parity never depends on these numbers (both read this file); they set
the physical scale of the rates (R21)."""
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SP = ["H2", "O2", "H2O", "H", "O", "OH", "HO2", "H2O2", "N2"]

# (reactants, products, type, k (A, b, Ea kJ/mol), k0 (falloff), troe (a, T***, T*, T**), efficiencies)
R = [
    ({"H": 1, "O2": 1}, {"OH": 1, "O": 1}, "elem", (3.52e16, -0.7, 71.42), None, None, None),
    ({"H2": 1, "O": 1}, {"OH": 1, "H": 1}, "elem", (5.06e4, 2.67, 26.32), None, None, None),
    ({"H2": 1, "OH": 1}, {"H2O": 1, "H": 1}, "elem", (1.17e9, 1.3, 15.21), None, None, None),
    ({"H": 1, "O2": 1}, {"HO2": 1}, "falloff", (4.65e12, 0.44, 0.0), (5.75e19, -1.4, 0.0),
     (0.5, 1e-30, 1e30, None), {"H2": 2.5, "H2O": 16.0}),
    ({"HO2": 1, "H": 1}, {"OH": 2}, "elem", (7.08e13, 0.0, 1.23), None, None, None),
    ({"HO2": 1, "H": 1}, {"H2": 1, "O2": 1}, "elem", (1.66e13, 0.0, 3.44), None, None, None),
    ({"HO2": 1, "OH": 1}, {"H2O": 1, "O2": 1}, "elem", (2.89e13, 0.0, -2.08), None, None, None),
    ({"H": 1, "OH": 1}, {"H2O": 1}, "threebody", (4.00e22, -2.0, 0.0), None, None, {"H2": 2.5, "H2O": 12.0}),
    ({"H": 2}, {"H2": 1}, "threebody", (1.30e18, -1.0, 0.0), None, None, {"H2": 2.5, "H2O": 12.0}),
    ({"HO2": 2}, {"H2O2": 1, "O2": 1}, "elem", (3.02e12, 0.0, 5.8), None, None, None),
    ({"HO2": 1, "H2": 1}, {"H2O2": 1, "H": 1}, "elem", (1.62e11, 0.61, 100.14), None, None, None),
    ({"H2O2": 1}, {"OH": 2}, "falloff", (2.62e19, -1.39, 214.74), (8.15e23, -1.9, 207.62),
     (0.735, 94.0, 1756.0, 5182.0), {"H2": 2.0, "H2O": 6.0}),
]
TYPES = {"elem": 0, "threebody": 1, "falloff": 2}


def si_A(A, order):  # (cm^3/mol)^(order-1)/s -> (m^3/kmol)^(order-1)/s; 1 cm^3/mol = 1e-3 m^3/kmol
    return A * 1e-3 ** (order - 1)


def main():
    out = {"name": "h2_9sp_kin", "species": SP, "units": "SI: A in (m^3/kmol)^(order-1)/s, Ea in J/kmol, T in K",
           "note": __doc__.split("\n\n")[1].replace("\n", " "), "reactions": []}
    for reac, prod, typ, k, k0, troe, eff in R:
        order = sum(reac.values())
        nu_f = [reac.get(s, 0) for s in SP]
        nu_r = [prod.get(s, 0) for s in SP]
        kinf_order = order + (1 if typ == "threebody" else 0)
        r = {"nu_f": nu_f, "nu_r": nu_r, "type": TYPES[typ], "reversible": 1,
             "A": si_A(k[0], kinf_order), "b": k[1], "Ea": k[2] * 1e6,
             "eff": [(eff or {}).get(s, 1.0) for s in SP]}
        if typ == "falloff":
            r.update(A0=si_A(k0[0], order + 1), b0=k0[1], Ea0=k0[2] * 1e6,
                     troe=[troe[0], troe[1], troe[2], troe[3] if troe[3] is not None else 1e30])
        else:
            r.update(A0=0.0, b0=0.0, Ea0=0.0, troe=[-1.0, 0.0, 0.0, 0.0])
        out["reactions"].append(r)
    path = os.path.join(ROOT, "data", "mech", "h2_9sp_kin.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print("wrote", path)


if __name__ == "__main__":
    main()
