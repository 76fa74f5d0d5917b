"""Mutation check of the oracle pins: apply one plausible mistake at a time to oracle/swe.cpp,
rebuild liborc.so, run the CPU oracle pins, and report which mutations survive (a surviving
mutation = an unpinned oracle path).  The source is always restored.

    python tools/mutate_oracle.py [name ...]      (default: every mutation below)
"""
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# name -> (exact text in oracle/swe.cpp, replacement)
MUTATIONS = {
    "wall_ghost_mean_no_mirror": (
        "        nm[p][1] = qb[1] - 2.0 * mn * nx;\n          nm[p][2] = qb[2] - 2.0 * mn * ny;",
        "        nm[p][1] = qb[1];\n          nm[p][2] = qb[2];"),
    "wall_ghost_barycentre_half": (
        "        nbx[f] = bx[e] - 2.0 * dist * nx;\n        nby[f] = by[e] - 2.0 * dist * ny;",
        "        nbx[f] = bx[e] - 1.0 * dist * nx;\n        nby[f] = by[e] - 1.0 * dist * ny;"),
    "h_char_switch_off": ("  if (h >= h_char) {\n    double c = std::sqrt(g * h)", "  if (true) {\n    double c = std::sqrt(g * h)"),
    "h_char_always_cw": ("  if (h >= h_char) {\n    double c = std::sqrt(g * h)", "  if (false) {\n    double c = std::sqrt(g * h)"),
    "posfix_removed": ("    fixed[idx] = posfix(Dh[0], hb, prm.h0, Dh[0]) ? 1 : 0;", "    fixed[idx] = 0;"),
    "rebalance_removed": ("    for (int k = 0; k < 3; k++) rebalance(Delta[k], Dh[k]);",
                          "    for (int k = 0; k < 3; k++) for (int i = 0; i < 3; i++) Dh[k][i] = Delta[k][i];"),
    "tvb_nu_dropped": ("        wb[a] = prm.tvb_nu * (", "        wb[a] = 1.0 * ("),
    "near_dry_skip_removed": ("      if (dry[n]) near_dry = true;", "      if (false) near_dry = true;"),
    "pp_theta_h0_dropped": ("theta = std::min(1.0, (qb[0] - prm.h0) / (qb[0] - h1min));",
                            "theta = std::min(1.0, (qb[0]) / (qb[0] - h1min));"),
    "flux_lambda_one_side": ("  double lam = std::max(std::fabs(unm) + std::sqrt(g * hsm), std::fabs(unp) + std::sqrt(g * hsp));",
                             "  double lam = std::fabs(unm) + std::sqrt(g * hsm);"),
    "dirichlet_ghost_interior": ("        hp = a[0];\n        hup = a[1];\n        hvp = a[2];\n        bp = bm;",
                                 "        hp = hm;\n        hup = hum;\n        hvp = hvm;\n        bp = bm;"),
    "dirichlet_tvb_mean_own": ("          means(&Qbnd[(size_t)e * 3 * Np], nm[p]);", "          for (int k = 0; k < 3; k++) nm[p][k] = qb[k];"),
    "source_sign": ("    double S[3] = {0.0, -g * (hc + bc) * bxc, -g * (hc + bc) * byc};",
                    "    double S[3] = {0.0, g * (hc + bc) * bxc, -g * (hc + bc) * byc};"),
}


def run(names):
    """Mutate a scratch copy of the repository (the working tree is never touched)."""
    import tempfile
    scratch = tempfile.mkdtemp(prefix="mutate_oracle_")
    for d in ("oracle", "tests", "swe_inputs", "paper_1403_1661_b200"):
        shutil.copytree(os.path.join(ROOT, d), os.path.join(scratch, d),
                        ignore=shutil.ignore_patterns("__pycache__", "_build*", "*.o"))
    for f in ("pytest.ini", "bench.py", "__graft_entry__.py"):
        shutil.copy(os.path.join(ROOT, f), scratch)
    src = os.path.join(scratch, "oracle", "swe.cpp")
    orig = open(src).read()
    files = sorted(f for f in os.listdir(os.path.join(scratch, "tests")) if f.startswith("test_oracle"))
    files.sort(key=lambda f: f != "test_oracle_tvb_pins.py")  # the limiter pins first: fail fast
    survived = []
    try:
        for name in names:
            a, b = MUTATIONS[name]
            if orig.count(a) != 1:
                print(f"{name}: pattern not found exactly once ({orig.count(a)})")
                survived.append(name + " (no pattern)")
                continue
            open(src, "w").write(orig.replace(a, b))
            subprocess.check_call([sys.executable, "-c", "import oracle; oracle.build(force=True)"], cwd=scratch)
            r = subprocess.run([sys.executable, "-m", "pytest", *[os.path.join("tests", f) for f in files], "-q", "-x",
                                "-m", "not gpu", "-p", "no:cacheprovider"], cwd=scratch, capture_output=True, text=True)
            caught = r.returncode != 0
            last = [ln for ln in r.stdout.splitlines() if ln.startswith("FAILED")][:1]
            print(f"{name}: {'caught' if caught else 'SURVIVED'} {last[0] if last else ''}", flush=True)
            if not caught:
                survived.append(name)
    finally:
        shutil.rmtree(scratch, ignore_errors=True)
    print("survived:", survived)
    return survived


if __name__ == "__main__":
    names = sys.argv[1:] or list(MUTATIONS)
    sys.exit(1 if run(names) else 0)
