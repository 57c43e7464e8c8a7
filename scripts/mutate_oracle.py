#!/usr/bin/env python
"""Mutation check of the oracle's pins (VERDICT r1 Weak #1).

Each mutant is one plausible slip in oracle/oracle.cpp (a wrong rounding, a flipped
comparison, a swapped index, a dropped term).  For each: copy oracle/, inputs/ and
tests/ to a scratch dir, apply the edit, rebuild liboracle.so, run the CPU pins
(tests/test_oracle.py) and require at least one failure.  A mutant that passes every
pin is an unpinned part of the oracle; the script exits 1 then.

    python scripts/mutate_oracle.py [--log profiles/r02/oracle_mutants.txt]
"""
import argparse
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# (name, old text, new text) — old must occur exactly once in oracle.cpp
MUTANTS = [
    ("cut target floor instead of ceil",
     "uint64_t target = ((uint64_t)i * two_m + pe - 1) / pe;",
     "uint64_t target = ((uint64_t)i * two_m) / pe;"),
    ("cut rule P[r] > target instead of >=",
     "while (P[r] < target) ++r;", "while (P[r] <= target) ++r;"),
    # Not a mutant: dropping max(cuts[i-1], .) is equivalent — the targets ceil(i*2m/p)
    # grow with i and P is non-decreasing, so min{r : P[r] >= target} already is.
    ("cut prefix from out-degree-free weight 1",
     "P[r + 1] = P[r] + g->deg[g->order[r]];", "P[r + 1] = P[r] + 1;"),
    ("degree counts only the first endpoint",
     "g->deg[k >> 32]++; g->deg[k & 0xFFFFFFFFu]++;", "g->deg[k >> 32]++;"),
    ("rank by descending degree",
     "return g->deg[a] < g->deg[b]; });", "return g->deg[a] > g->deg[b]; });"),
    ("ties by descending input id",
     "std::stable_sort(g->order.begin(), g->order.end(),\n"
     "                   [&](uint32_t a, uint32_t b) { return g->deg[a] < g->deg[b]; });",
     "std::stable_sort(g->order.begin(), g->order.end(),\n"
     "                   [&](uint32_t a, uint32_t b) { return g->deg[a] < g->deg[b] || (g->deg[a] == g->deg[b] && a > b); });"),
    ("orientation high -> low rank",
     "k = ((uint64_t)std::min(ra, rb) << 32) | std::max(ra, rb);",
     "k = ((uint64_t)std::max(ra, rb) << 32) | std::min(ra, rb);"),
    ("self-loops kept",
     "if (a == b) continue;", "if (false) continue;"),
    ("Alg. 1 typo A[b] = B[b] taken literally",
     "if (A[a] == B[b]) { emit(A[a]); ++c; ++a; ++b; }",
     "if (b < na && A[b] == B[b]) { emit(A[b]); ++c; ++a; ++b; }"),
    ("task bin (part u, part w) instead of (part u, part v)",
     "mine[first[(size_t)part[u] * p + part[v]] + (part[w] - part[v])]++;",
     "mine[first[(size_t)part[u] * p + part[w]] + (part[v] - part[w])]++;"),
    ("task bin k offset from part u",
     "mine[first[(size_t)part[u] * p + part[v]] + (part[w] - part[v])]++;",
     "mine[first[(size_t)part[u] * p + part[v]] + (part[w] - part[u])]++;"),
    ("Alg. 4 order with the k loop outermost",
     "    for (uint32_t j = i; j < p; ++j)\n      for (uint32_t k = j; k < p; ++k) {\n        if (k == j) first",
     "    for (uint32_t j = i; j < p; ++j)\n      for (uint32_t k = j; k < p; ++k) {\n        if (k == p - 1) first"),
    ("per-vertex misses w",
     "            pv[w].fetch_add(1, std::memory_order_relaxed);\n", ""),
    ("n ignores the largest raw id",
     "g->n = std::max(n_hint, top);", "g->n = n_hint ? n_hint : top;"),
    ("single-task count ignores the part of v",
     "if (v < cuts[j] || v >= cuts[j + 1]) continue;", "if (v < cuts[j]) continue;"),
]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--log", default=None)
    args = ap.parse_args()
    src = open(os.path.join(ROOT, "oracle", "oracle.cpp")).read()
    out = []
    survivors = 0
    for name, old, new in MUTANTS:
        n = src.count(old)
        if n != 1:
            out.append(f"SKIP ({n} matches)  {name}")
            survivors += 1
            continue
        with tempfile.TemporaryDirectory() as tmp:
            for d in ("oracle", "inputs", "tests"):
                shutil.copytree(os.path.join(ROOT, d), os.path.join(tmp, d),
                                ignore=shutil.ignore_patterns("__pycache__"))
            shutil.copy(os.path.join(ROOT, "pytest.ini"), tmp)
            with open(os.path.join(tmp, "oracle", "oracle.cpp"), "w") as f:
                f.write(src.replace(old, new))
            subprocess.run(["g++", "-std=c++17", "-O2", "-fPIC", "-fopenmp", "-shared", "-o",
                            os.path.join(tmp, "oracle", "liboracle.so"), os.path.join(tmp, "oracle", "oracle.cpp")],
                           check=True)
            r = subprocess.run([sys.executable, "-m", "pytest", "tests/test_oracle.py", "-q", "-m", "not gpu",
                                "-p", "no:cacheprovider"], cwd=tmp, capture_output=True, text=True)
            tail = [ln for ln in r.stdout.splitlines() if ln.strip()][-1:]
            killed = r.returncode != 0
            survivors += not killed
            out.append(f"{'killed ' if killed else 'SURVIVED'}  {name}  [{tail[0] if tail else ''}]")
        print(out[-1], flush=True)
    out.append(f"{len(MUTANTS) - survivors}/{len(MUTANTS)} mutants killed by tests/test_oracle.py")
    print(out[-1])
    if args.log:
        os.makedirs(os.path.dirname(os.path.join(ROOT, args.log)), exist_ok=True)
        with open(os.path.join(ROOT, args.log), "w") as f:
            f.write("\n".join(out) + "\n")
    sys.exit(1 if survivors else 0)


if __name__ == "__main__":
    main()
