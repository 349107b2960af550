"""Mutation check of the oracle's pins: each mutant is the oracle's C
source with one plausible mistake (a dropped term, a wrong operand, an off-by-one), built to a
temporary library; the CPU pin suite (tests/test_oracle_pins.py) must fail on every mutant and
pass on the unmodified source. Writes profiles/r02_oracle_mutations.json.

    python tools/oracle_mutation_check.py
"""
import json
import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "oracle", "wmd_oracle.c")

# (name, exact text in wmd_oracle.c, replacement)
MUTANTS = [
    ("sqrt dropped from the distance", "  return sqrt(s);\n}", "  return s;\n}"),
    ("M squared inside exp", "double kk = exp(-lambda * m);", "double kk = exp(-lambda * m * m);"),
    ("1/r dropped from p = (1/r) K", "p[(int64_t)i * V + k] = (1.0 / r[i]) * kk;", "p[(int64_t)i * V + k] = kk;"),
    ("x0 perturbed in one query row", "for (int64_t q = 0; q < (int64_t)v_r * N; ++q) x[q] = 1.0 / (double)v_r;",
     "for (int64_t q = 0; q < (int64_t)v_r * N; ++q) x[q] = (q % v_r == 0 ? 1.001 : 1.0) / (double)v_r;"),
    ("c dropped in the SDDMM", "          v[e] = (double)val[e] * (1.0 / s);\n        }\n      }\n      for (int32_t i = 0; i < v_r; ++i) {",
     "          v[e] = 1.0 / s;\n        }\n      }\n      for (int32_t i = 0; i < v_r; ++i) {"),
    ("one extra x-update", "for (; it < max_iter; ++it) {", "for (; it <= max_iter; ++it) {"),
    ("u dropped from the final sum", "for (int64_t e = b; e < en; ++e) s += KM[(int64_t)i * V + row_idx[e]] * v[e];\n      w += u[i] * s;",
     "for (int64_t e = b; e < en; ++e) s += KM[(int64_t)i * V + row_idx[e]] * v[e];\n      w += s;"),
    ("K instead of K.*M in the final step", "for (int64_t e = b; e < en; ++e) s += KM[(int64_t)i * V + row_idx[e]] * v[e];\n      w += u[i] * s;",
     "for (int64_t e = b; e < en; ++e) s += K[(int64_t)i * V + row_idx[e]] * v[e];\n      w += u[i] * s;"),
]


def run_pins(lib):
    env = dict(os.environ, WMD_ORACLE_LIB_OVERRIDE=lib) if lib else dict(os.environ)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                        os.path.join(ROOT, "tests", "test_oracle_pins.py")],
                       cwd=ROOT, env=env, capture_output=True, text=True)
    last = [l for l in r.stdout.strip().splitlines() if l.strip()][-1:]
    return r.returncode, (last[0] if last else "")


def main():
    src = open(SRC).read()
    out = {"unmodified": None, "mutants": []}
    rc, tail = run_pins(None)
    out["unmodified"] = {"pins_pass": rc == 0, "summary": tail}
    with tempfile.TemporaryDirectory() as tmp:
        for i, (name, old, new) in enumerate(MUTANTS):
            assert src.count(old) == 1, f"mutation site not unique / missing: {name}"
            path = os.path.join(tmp, f"m{i}.c")
            with open(path, "w") as f:
                f.write(src.replace(old, new))
            lib = os.path.join(tmp, f"m{i}.so")
            subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-fno-fast-math",
                                   "-ffp-contract=off", "-o", lib, path, "-lm"])
            rc, tail = run_pins(lib)
            out["mutants"].append({"mutation": name, "caught": rc != 0, "summary": tail})
            print(f"{name:45s} caught={rc != 0}  {tail}", flush=True)
    out["all_caught"] = all(m["caught"] for m in out["mutants"])
    with open(os.path.join(ROOT, "profiles", "r02_oracle_mutations.json"), "w") as f:
        json.dump(out, f, indent=1)
        f.write("\n")
    print("unmodified pins pass:", out["unmodified"]["pins_pass"], " all mutants caught:", out["all_caught"])
    return 0 if out["all_caught"] and out["unmodified"]["pins_pass"] else 1


if __name__ == "__main__":
    sys.exit(main())
