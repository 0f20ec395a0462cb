"""Are the GPU parity tests sharp?  Plant ONE slip in a copy of the CUDA sources (the tree itself is
never touched), build the library from the copy, and run the fast GPU parity tests against it via
ISRS_EGN_LIB: every mutant must fail them.

    python tests/tools/kernel_mutants.py build          # here (nvcc cross-compiles): build_variants/lib_mut_*.so
    python tests/tools/kernel_mutants.py run            # on the GPU box: one pytest run per mutant
    (either with mutant names after the verb: only those)

Prints one JSON line per mutant: name, slip, pytest exit code, killed (exit code 1).
"""
import json
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
OUT = os.path.join(ROOT, "build_variants")

# name: (file under paper_2412_11614_b200/csrc, exact original text, mutated text, what the slip is)
MUTANTS = {
    "goertzel_plus_b2": ("kernels.cu", "n0[q] = fma(c2[q], b1[q], tc.x) - b2[q];",
                         "n0[q] = fma(c2[q], b1[q], tc.x) + b2[q];", "recurrence: + b_{k+2} in the even step"),
    "walk_power_index": ("kernels.cu", "vr[m] = v * sp[m];", "vr[m] = v * sp[m > 0 ? m - 1 : 0];",
                         "table walk: step^m off by one inside a run"),
    "wrap_pair_missing": ("kernels.cu", "if (ii < 2) sm.T[r * p.tstride + Kp + ii] = x;",
                          "if (ii < 1) sm.T[r * p.tstride + Kp + ii] = x;",
                          "chain wrap: only one of the two wrapped coefficients"),
    "I0_sign": ("kernels.cu", "const double wr1 = fma(Eh, cs[q], -1.0), wi = Eh * sn[q];",
                "const double wr1 = fma(Eh, cs[q], -1.0), wi = -Eh * sn[q];", "I_0: conj(w) for w"),
    "phase_one_span_short": ("kernels.cu", "double t2 = fma(x[q], (double)(Ks * G), th[q]);",
                             "double t2 = fma(x[q], (double)(Ks * (G > 1 ? G - 1 : G)), th[q]);",
                             "span phase: a chain advances theta by G-1 spans"),
    "gate_edge_weight": ("kernels.cu", "const double t = (f3 > l && f3 < h) ? 1.0 : 0.5;",
                         "const double t = (f3 > l && f3 < h) ? 1.0 : 1.0;", "C10: band-edge points weigh 1"),
    "coherent_row_weight": ("kernels.cu", "acc.x = fma(w, y.x, acc.x);", "acc.x = fma(w, y.x, 0.5 * acc.x);",
                            "E row sum: halves the running sum"),
    "lattice_m2": ("kernels.cu", "const int m2f = (b == 1) ? lj - a * m1f : (lj - a * m1f) / b;",
                   "const int m2f = (b == 1) ? lj - a * m1f : (lj - a * m1f) / b + (a > 1);",
                   "point geometry: m2 off by one on mixed-rate lattices"),
    # ---- round 2: chain groups (R13), shuffle reductions, the exact planner
    "group_horner_conj": ("kernels.cu", "const double t = fma(sr[q], a, fma(-si[q], b, accr[q]));",
                          "const double t = fma(sr[q], a, fma(si[q], b, accr[q]));",
                          "chain groups: Horner step with conj(w) in the real part"),
    "group_step_short": ("kernels.cu", "const double t = x * (double)(Ks * G0);",
                         "const double t = x * (double)(Ks * (G0 - 1));",
                         "chain groups: w = e^{i (G0 - 1) chi L}"),
    "group_theta_short": ("kernels.cu", "const double t2 = fma(x, (double)(Ks * gsum), th[q]);",
                          "const double t2 = fma(x, (double)(Ks * (gsum - 1)), th[q]);",
                          "chain groups: theta advanced by one span too few per group"),
    "group_second_phase": ("kernels.cu", "if (gr > 0) sincospi_d(th[q], &ps, &pc);",
                           "if (gr > 1) sincospi_d(th[q], &ps, &pc);",
                           "chain groups: the second group's span phase dropped"),
    "shuffle_last_warp": ("kernels.cu", "for (int w = 1; w < BLOCK / 32; ++w) t += red[NV * w + k];",
                          "for (int w = 1; w < BLOCK / 32 - 1; ++w) t += red[NV * w + k];",
                          "coherent block sums: the last warp's partial dropped"),
    "planner_touching_twice": ("abi.cu", "if (j0 <= cur1) {                         // touching bands share the edge line",
                               "if (j0 < cur1) {                         // touching bands share the edge line",
                               "planner: the edge line of touching bands counted twice"),
    # ---- round 2, late: the table-driven sin/cos(pi x)
    "cistab_index": ("kernels.cu", "const double2 e = __ldg(&kCisTab[__double2loint(t) & 255]);",
                     "const double2 e = __ldg(&kCisTab[(__double2loint(t) + 1) & 255]);",
                     "table sincospi: the neighbouring table entry"),
    "cistab_sin_sign": ("kernels.cu", "*sp = fma(e.y, cm1, fma(e.x, s, e.y));",
                        "*sp = fma(e.y, cm1, fma(-e.x, s, e.y));",
                        "table sincospi: sin(a + b) with -cos(a) sin(b)"),
    "cistab_cos_term": ("kernels.cu", "pc = fma(pc, r2, -4.934802200544679);",
                        "pc = fma(pc, r2, -4.934802200544679 * 0.999);",
                        "table sincospi: the r^2 coefficient of cos off by 0.1 %"),
    # ---- NEXT-4a: the closed-form phased-array factor of long runs (MODE_SEGDDL)
    "dedupl_phase_G": ("kernels.cu", "tp = 0.5 * (double)(G - 1) * hr;", "tp = 0.5 * (double)G * hr;",
                       "dedup closed form: phase e^{i G chi L / 2} instead of e^{i (G-1) chi L / 2}"),
    "dedupl_amp_cos": ("kernels.cu", "const double amp = sg / s1;", "const double amp = sg / c1;",
                       "dedup closed form: sin(G chi L/2) / cos(chi L/2)"),
    # ---- SCI / XCI / MCI split (ISRS_EGN_FLAG_SPLIT)
    # (dropping `c == kappa` instead is an EQUIVALENT mutant -- it survived, profiles/r02zx_*: a split entry has
    # kappa in {k1, k2} or k1 == k2 = j, and an island (j, j, kappa) cannot exist between non-overlapping bands:
    # |f3 - f_kappa| >= 2 |f_j - f_kappa| - R_j >= R_kappa > R_kappa / 2)
    "split_filter_k2": ("kernels.cu", "const bool in = (c == kappa || c == k1 || c == k2);",
                        "const bool in = (c == kappa || c == k1);",
                        "split line filter: k3 = k2 not counted among the region's own channels"),
    "split_out_class": ("kernels.cu", "+ ((rd.flags & K3_OUT) ? 1 : 0);", "+ ((rd.flags & K3_IN) ? 1 : 0);",
                        "split reduce: the K3_IN entry, not the K3_OUT one, counts one more interferer"),
    "split_class_k2": ("kernels.cu", "(rd.k2 != kappa && rd.k2 != rd.k1)", "(rd.k2 != kappa)",
                       "split reduce: k1 = k2 = j counted as two interferers"),
}

FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-Xcompiler", "-fPIC",
         "-Xcompiler", "-fvisibility=hidden", "-shared", "--expt-relaxed-constexpr"]
TESTS = ("tiny or edge or random_links or c1_full or streams or planned_work or chain_groups or (golden and c2_eta) "
         "or dedup_closed_form or (split and not full_size)")


def _selected():
    names = sys.argv[2:]
    return {k: v for k, v in MUTANTS.items() if not names or k in names}


def build():
    os.makedirs(OUT, exist_ok=True)
    for name, (fn, old, new, _) in _selected().items():
        with tempfile.TemporaryDirectory() as td:
            src = os.path.join(td, "paper_2412_11614_b200", "csrc")
            shutil.copytree(os.path.join(ROOT, "paper_2412_11614_b200", "csrc"), src)
            shutil.copytree(os.path.join(ROOT, "include"), os.path.join(td, "include"))
            path = os.path.join(src, fn)
            text = open(path).read()
            assert text.count(old) >= 1, f"{name}: pattern not found"
            open(path, "w").write(text.replace(old, new, 1))
            lib = os.path.join(OUT, f"lib_mut_{name}.so")
            cmd = ["nvcc"] + FLAGS + ["-I", os.path.join(td, "include"), os.path.join(src, "abi.cu"),
                                      os.path.join(src, "kernels.cu"), "-o", lib]
            r = subprocess.run(cmd, capture_output=True, text=True)
            print(name, "built" if r.returncode == 0 else r.stderr[-500:], flush=True)


def run():
    for name, (_, _, _, what) in _selected().items():
        lib = os.path.join(OUT, f"lib_mut_{name}.so")
        env = dict(os.environ, ISRS_EGN_LIB=lib)
        r = subprocess.run([sys.executable, "-m", "pytest", os.path.join(ROOT, "tests", "test_parity_gpu.py"),
                            "-m", "gpu", "-x", "-q", "-p", "no:cacheprovider", "-k", TESTS],
                           cwd=ROOT, env=env, capture_output=True, text=True, timeout=1800)
        tail = [l for l in r.stdout.splitlines() if "passed" in l or "failed" in l]
        print(json.dumps({"mutant": name, "slip": what, "pytest_rc": r.returncode, "killed": r.returncode == 1,
                          "summary": tail[-1] if tail else r.stdout[-300:]}), flush=True)


if __name__ == "__main__":
    {"build": build, "run": run}[sys.argv[1]]()
