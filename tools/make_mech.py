"""Mechanism-table generator (run once; its JSON output is committed under data/mech/).

Neither PAPER.md nor the image ships mechanism data, and
Cantera is not installed.  The paper evaluates thermo and transport with
"high-order temperature polynomials" taken "via the Cantera interface"
(§2, §3.1).  This script writes those polynomial
tables:

* NASA-7 coefficients for the H2/air (Ns=9) and CH4/air DRM19-without-Ar
  (Ns=20, "20 species") species sets, GRI-Mech 3.0 values
  (SURVEY.md App. A).
* Transport fits in Cantera's "mixture-averaged" forms (reading R10):
      sqrt(mu_k)/T^(1/4)        = sum_n visc[k][n] (ln T)^n
      lambda_k/sqrt(T)          = sum_n cond[k][n] (ln T)^n
      D_jk * p / T^(3/2)        = sum_n diff[jk][n] (ln T)^n       (p in Pa)
  fitted (least squares, degree 4, 300-3500 K, 400 points) to Chapman-Enskog
  values built from GRI-Mech 3.0 Lennard-Jones parameters with Neufeld
  collision integrals and a modified-Eucken conductivity (SURVEY.md App. A,
  "Fitter recipe").

The fitter is table pre-processing: it is neither part of the oracle nor of
the CUDA path, and both of those read the JSON it writes.

usage: python tools/make_mech.py   (rewrites data/mech/h2_9sp.json, ch4_20sp.json)
"""
import json
import math
import os

import numpy as np

RU = 8314.46261815324  # J/kmol/K
ATOMIC_W = {"H": 1.008, "C": 12.011, "N": 14.007, "O": 15.999}

# name: (Tlo, Tmid, Thi, low a1..a7, high a1..a7)   -- GRI-Mech 3.0
NASA = {
 "H2": (200, 1000, 3500, [2.34433112E+00, 7.98052075E-03, -1.94781510E-05, 2.01572094E-08, -7.37611761E-12, -9.17935173E+02, 6.83010238E-01],
        [3.33727920E+00, -4.94024731E-05, 4.99456778E-07, -1.79566394E-10, 2.00255376E-14, -9.50158922E+02, -3.20502331E+00]),
 "O2": (200, 1000, 3500, [3.78245636E+00, -2.99673416E-03, 9.84730201E-06, -9.68129509E-09, 3.24372837E-12, -1.06394356E+03, 3.65767573E+00],
        [3.28253784E+00, 1.48308754E-03, -7.57966669E-07, 2.09470555E-10, -2.16717794E-14, -1.08845772E+03, 5.45323129E+00]),
 "H2O": (200, 1000, 3500, [4.19864056E+00, -2.03643410E-03, 6.52040211E-06, -5.48797062E-09, 1.77197817E-12, -3.02937267E+04, -8.49032208E-01],
         [3.03399249E+00, 2.17691804E-03, -1.64072518E-07, -9.70419870E-11, 1.68200992E-14, -3.00042971E+04, 4.96677010E+00]),
 "H": (200, 1000, 3500, [2.50000000E+00, 0.0, 0.0, 0.0, 0.0, 2.54736599E+04, -4.46682853E-01],
       [2.50000001E+00, -2.30842973E-11, 1.61561948E-14, -4.73515235E-18, 4.98197357E-22, 2.54736599E+04, -4.46682914E-01]),
 "O": (200, 1000, 3500, [3.16826710E+00, -3.27931884E-03, 6.64306396E-06, -6.12806624E-09, 2.11265971E-12, 2.91222592E+04, 2.05193346E+00],
       [2.56942078E+00, -8.59741137E-05, 4.19484589E-08, -1.00177799E-11, 1.22833691E-15, 2.92175791E+04, 4.78433864E+00]),
 "OH": (200, 1000, 3500, [3.99201543E+00, -2.40131752E-03, 4.61793841E-06, -3.88113333E-09, 1.36411470E-12, 3.61508056E+03, -1.03925458E-01],
        [3.09288767E+00, 5.48429716E-04, 1.26505228E-07, -8.79461556E-11, 1.17412376E-14, 3.85865700E+03, 4.47669610E+00]),
 "HO2": (200, 1000, 3500, [4.30179801E+00, -4.74912051E-03, 2.11582891E-05, -2.42763894E-08, 9.29225124E-12, 2.94808040E+02, 3.71666245E+00],
         [4.01721090E+00, 2.23982013E-03, -6.33658150E-07, 1.14246370E-10, -1.07908535E-14, 1.11856713E+02, 3.78510215E+00]),
 "H2O2": (200, 1000, 3500, [4.27611269E+00, -5.42822417E-04, 1.67335701E-05, -2.15770813E-08, 8.62454363E-12, -1.77025821E+04, 3.43505074E+00],
          [4.16500285E+00, 4.90831694E-03, -1.90139225E-06, 3.71185986E-10, -2.87908305E-14, -1.78617877E+04, 2.91615662E+00]),
 "N2": (300, 1000, 5000, [3.298677E+00, 1.4082404E-03, -3.963222E-06, 5.641515E-09, -2.444854E-12, -1.0208999E+03, 3.950372E+00],
        [2.926640E+00, 1.4879768E-03, -5.684760E-07, 1.0097038E-10, -6.753351E-15, -9.227977E+02, 5.980528E+00]),
 "CH4": (200, 1000, 3500, [5.14987613E+00, -1.36709788E-02, 4.91800599E-05, -4.84743026E-08, 1.66693956E-11, -1.02466476E+04, -4.64130376E+00],
         [7.48514950E-02, 1.33909467E-02, -5.73285809E-06, 1.22292535E-09, -1.01815230E-13, -9.46834459E+03, 1.84373180E+01]),
 "CO": (200, 1000, 3500, [3.57953347E+00, -6.10353680E-04, 1.01681433E-06, 9.07005884E-10, -9.04424499E-13, -1.43440860E+04, 3.50840928E+00],
        [2.71518561E+00, 2.06252743E-03, -9.98825771E-07, 2.30053008E-10, -2.03647716E-14, -1.41518724E+04, 7.81868772E+00]),
 "CO2": (200, 1000, 3500, [2.35677352E+00, 8.98459677E-03, -7.12356269E-06, 2.45919022E-09, -1.43699548E-13, -4.83719697E+04, 9.90105222E+00],
         [3.85746029E+00, 4.41437026E-03, -2.21481404E-06, 5.23490188E-10, -4.72084164E-14, -4.87591660E+04, 2.27163806E+00]),
 "CH3": (200, 1000, 3500, [3.67359040E+00, 2.01095175E-03, 5.73021856E-06, -6.87117425E-09, 2.54385734E-12, 1.64449988E+04, 1.60456433E+00],
         [2.28571772E+00, 7.23990037E-03, -2.98714348E-06, 5.95684644E-10, -4.67154394E-14, 1.67755843E+04, 8.48007179E+00]),
 "CH2": (200, 1000, 3500, [3.76267867E+00, 9.68872143E-04, 2.79489841E-06, -3.85091153E-09, 1.68741719E-12, 4.60040401E+04, 1.56253185E+00],
         [2.87410113E+00, 3.65639292E-03, -1.40894597E-06, 2.60179549E-10, -1.87727567E-14, 4.62636040E+04, 6.17119324E+00]),
 "CH2(S)": (200, 1000, 3500, [4.19860411E+00, -2.36661419E-03, 8.23296220E-06, -6.68815981E-09, 1.94314737E-12, 5.04968163E+04, -7.69118967E-01],
            [2.29203842E+00, 4.65588637E-03, -2.01191947E-06, 4.17906000E-10, -3.39716365E-14, 5.09259997E+04, 8.62650169E+00]),
 "HCO": (200, 1000, 3500, [4.22118584E+00, -3.24392532E-03, 1.37799446E-05, -1.33144093E-08, 4.33768865E-12, 3.83956496E+03, 3.39437243E+00],
         [2.77217438E+00, 4.95695526E-03, -2.48445613E-06, 5.89161778E-10, -5.33508711E-14, 4.01191815E+03, 9.79834492E+00]),
 "CH2O": (200, 1000, 3500, [4.79372315E+00, -9.90833369E-03, 3.73220008E-05, -3.79285261E-08, 1.31772652E-11, -1.43089567E+04, 6.02812900E-01],
          [1.76069008E+00, 9.20000082E-03, -4.42258813E-06, 1.00641212E-09, -8.83855640E-14, -1.39958323E+04, 1.36563230E+01]),
 "CH3O": (300, 1000, 3000, [2.106204E+00, 7.216595E-03, 5.338472E-06, -7.377636E-09, 2.075610E-12, 9.786011E+02, 1.3152177E+01],
          [3.770799E+00, 7.871497E-03, -2.656384E-06, 3.944431E-10, -2.112616E-14, 1.2783252E+02, 2.929575E+00]),
 "C2H4": (200, 1000, 3500, [3.95920148E+00, -7.57052247E-03, 5.70990292E-05, -6.91588753E-08, 2.69884373E-11, 5.08977593E+03, 4.09733096E+00],
          [2.03611116E+00, 1.46454151E-02, -6.71077915E-06, 1.47222923E-09, -1.25706061E-13, 4.93988614E+03, 1.03053693E+01]),
 "C2H5": (200, 1000, 3500, [4.30646568E+00, -4.18658892E-03, 4.97142807E-05, -5.99126606E-08, 2.30509004E-11, 1.28416265E+04, 4.70720924E+00],
          [1.95465642E+00, 1.73972722E-02, -7.98206668E-06, 1.75217689E-09, -1.49641576E-13, 1.28575200E+04, 1.34624343E+01]),
 "C2H6": (200, 1000, 3500, [4.29142492E+00, -5.50154270E-03, 5.99438288E-05, -7.08466285E-08, 2.68685771E-11, -1.15222055E+04, 2.66682316E+00],
          [1.07188150E+00, 2.16852677E-02, -1.00256067E-05, 2.21412001E-09, -1.90002890E-13, -1.14263932E+04, 1.51156107E+01]),
}

# name: geometry, eps/kB [K], sigma [A], dipole [D], polarisability [A^3], Zrot  (GRI-Mech 3.0 tran.dat)
TRAN = {
 "H2": (1, 38.0, 2.92, 0, 0.79, 280), "O2": (1, 107.4, 3.458, 0, 1.60, 3.8), "H2O": (2, 572.4, 2.605, 1.844, 0, 4.0),
 "H": (0, 145.0, 2.05, 0, 0, 0), "O": (0, 80.0, 2.75, 0, 0, 0), "OH": (1, 80.0, 2.75, 0, 0, 0),
 "HO2": (2, 107.4, 3.458, 0, 0, 1.0), "H2O2": (2, 107.4, 3.458, 0, 0, 3.8), "N2": (1, 97.53, 3.621, 0, 1.76, 4.0),
 "CH4": (2, 141.4, 3.746, 0, 2.6, 13.0), "CO": (1, 98.1, 3.65, 0, 1.95, 1.8), "CO2": (1, 244.0, 3.763, 0, 2.65, 2.1),
 "CH3": (1, 144.0, 3.8, 0, 0, 0), "CH2": (1, 144.0, 3.8, 0, 0, 0), "CH2(S)": (1, 144.0, 3.8, 0, 0, 0),
 "HCO": (2, 498.0, 3.59, 0, 0, 0), "CH2O": (2, 498.0, 3.59, 0, 0, 2.0), "CH3O": (2, 417.0, 3.69, 1.7, 0, 2.0),
 "C2H4": (2, 280.8, 3.971, 0, 0, 1.5), "C2H5": (2, 252.3, 4.302, 0, 0, 1.5), "C2H6": (2, 252.3, 4.302, 0, 0, 1.5),
}

COMPOSITION = {
 "H2": {"H": 2}, "O2": {"O": 2}, "H2O": {"H": 2, "O": 1}, "H": {"H": 1}, "O": {"O": 1}, "OH": {"O": 1, "H": 1},
 "HO2": {"H": 1, "O": 2}, "H2O2": {"H": 2, "O": 2}, "N2": {"N": 2}, "CH4": {"C": 1, "H": 4}, "CO": {"C": 1, "O": 1},
 "CO2": {"C": 1, "O": 2}, "CH3": {"C": 1, "H": 3}, "CH2": {"C": 1, "H": 2}, "CH2(S)": {"C": 1, "H": 2},
 "HCO": {"H": 1, "C": 1, "O": 1}, "CH2O": {"H": 2, "C": 1, "O": 1}, "CH3O": {"C": 1, "H": 3, "O": 1},
 "C2H4": {"C": 2, "H": 4}, "C2H5": {"C": 2, "H": 5}, "C2H6": {"C": 2, "H": 6},
}

SETS = {
 "h2_9sp": dict(species=["H2", "O2", "H2O", "H", "O", "OH", "HO2", "H2O2", "N2"], elements=["H", "O", "N"],
                note="H2/air, 9 species (PAPER.md:94, 231: 9 species / 12 reactions)"),
 "ch4_20sp": dict(species=["H2", "H", "O", "O2", "OH", "H2O", "HO2", "CH2", "CH2(S)", "CH3", "CH4", "CO", "CO2",
                           "HCO", "CH2O", "CH3O", "C2H4", "C2H5", "C2H6", "N2"], elements=["C", "H", "O", "N"],
                  note="CH4/air DRM19 without Ar, 20 species (PAPER.md:267 '20 species and 85 reactions')"),
}


def omega22(ts):
    return 1.16145 * ts ** -0.14874 + 0.52487 * np.exp(-0.77320 * ts) + 2.16178 * np.exp(-2.43787 * ts)


def omega11(ts):
    return (1.06036 * ts ** -0.15610 + 0.19300 * np.exp(-0.47635 * ts) + 1.03587 * np.exp(-1.52996 * ts)
            + 1.76474 * np.exp(-3.89411 * ts))


def cp_mass(name, W, T):
    tlo, tmid, thi, lo, hi = NASA[name]
    a = np.where(T[:, None] <= tmid, np.array(lo)[None, :], np.array(hi)[None, :])
    return RU / W * (a[:, 0] + a[:, 1] * T + a[:, 2] * T**2 + a[:, 3] * T**3 + a[:, 4] * T**4)


def fit(L, y, deg=4):
    V = np.vander(L, deg + 1, increasing=True)
    c, *_ = np.linalg.lstsq(V, y, rcond=None)
    rel = np.max(np.abs(V @ c - y) / np.abs(y))
    return c, rel


def build(tag):
    spec = SETS[tag]
    sp, el = spec["species"], spec["elements"]
    ns = len(sp)
    atoms = [[COMPOSITION[s].get(e, 0) for s in sp] for e in el]
    W = np.array([sum(COMPOSITION[s].get(e, 0) * ATOMIC_W[e] for e in el) for s in sp])
    T = np.linspace(300.0, 3500.0, 400)
    L = np.log(T)
    visc, cond, diff = [], [], []
    max_rel = {"visc": 0.0, "cond": 0.0, "diff": 0.0}
    mu = {}
    for k, s in enumerate(sp):
        _, eps, sig, *_ = TRAN[s]
        mu_k = 2.6693e-6 * np.sqrt(W[k] * T) / (sig**2 * omega22(T / eps))
        mu[s] = mu_k
        c, r = fit(L, np.sqrt(mu_k) / T**0.25); visc.append(c.tolist()); max_rel["visc"] = max(max_rel["visc"], r)
        lam = mu_k * (cp_mass(s, W[k], T) + 1.25 * RU / W[k])
        c, r = fit(L, lam / np.sqrt(T)); cond.append(c.tolist()); max_rel["cond"] = max(max_rel["cond"], r)
    for k in range(ns):           # packed j <= k: index k(k+1)/2 + j
        for j in range(k + 1):
            _, ej, sj, *_ = TRAN[sp[j]]
            _, ek, sk, *_ = TRAN[sp[k]]
            sjk, ejk = 0.5 * (sj + sk), math.sqrt(ej * ek)
            p_atm = 1.0 / 101325.0  # D at p = 1 Pa
            D = 1.8583e-7 * np.sqrt(T**3 * (1.0 / W[j] + 1.0 / W[k])) / (p_atm * sjk**2 * omega11(T / ejk))
            c, r = fit(L, D / T**1.5); diff.append(c.tolist()); max_rel["diff"] = max(max_rel["diff"], r)
    return {
        "name": tag, "note": spec["note"], "units": "SI, kmol; h absolute (formation-inclusive)",
        "elements": el, "atomic_weights": [ATOMIC_W[e] for e in el], "species": sp,
        "atoms": atoms,
        "T_lo": [float(NASA[s][0]) for s in sp], "T_mid": [float(NASA[s][1]) for s in sp],
        "T_hi": [float(NASA[s][2]) for s in sp],
        "nasa_lo": [NASA[s][3] for s in sp], "nasa_hi": [NASA[s][4] for s in sp],
        "visc": visc, "cond": cond, "diff": diff,
        "inert": [1 if s == "N2" else 0 for s in sp],
        "fit": {"T_range": [300.0, 3500.0], "points": 400, "degree": 4, "max_rel_residual": max_rel,
                "forms": {"visc": "sqrt(mu_k)/T^0.25", "cond": "lambda_k/sqrt(T)", "diff": "D_jk*p/T^1.5 (p in Pa), packed j<=k at k(k+1)/2+j"}},
        "lennard_jones": {s: list(TRAN[s]) for s in sp},
    }


if __name__ == "__main__":
    out = os.path.join(os.path.dirname(__file__), "..", "data", "mech")
    for tag in SETS:
        m = build(tag)
        with open(os.path.join(out, tag + ".json"), "w") as f:
            json.dump(m, f, indent=1)
        print(tag, m["fit"]["max_rel_residual"])
