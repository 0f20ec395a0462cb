"""ORACLE — test infrastructure only.

A plain, slow, obviously correct CPU implementation (numpy, fp64) of what the CUDA path
computes: the ISRS EGN NLI coefficient eta(f_COI) with the segment closed-form FWM
efficiency factor (Eqs. 7-10), plus the integral form (Eq. 23, `quad` mode) and
the Maclaurin closed form (Eq. 4) used as pins and for the NEXT rows.

Only `tests/` (including the whole-eta parity and oracle-timing scripts in `tests/tools/`),
`__graft_entry__.smoke()` and `bench.py`'s cpu_baseline / `--impl reference` legs may import
anything under `oracle/`.  The product package
`paper_2412_11614_b200/` never imports it, and this package never imports the product:
the two share no code.  The only shared module is `workloads/` (seeded inputs, no method
arithmetic).

Citations: `P:n` = /root/reference/PAPER.md line n (section/equation named beside it);
readings C1..C17 are the ambiguity ledger of SURVEY.md §8(c), restated in DESIGN.md.

Modules
  units    — datasheet conversions (independent of workloads/, pinned against it)
  formats  — Phi, Psi from constellation moments (reading C9)
  isrs     — L_eff, zeta, rho(z,f) Eq. 13/25, SRS gain Eq. 14, Delta-rho Eq. 12
  fwm      — chi Eq. 5, GN eta Eq. 6, segment mu Eqs. 8-10, Maclaurin mu Eq. 4, quad mu Eq. 23
  link     — link function Y, Eq. 22 (reading C3; the literal gain products, NEXT-4b / R11)
  egn      — canonicalisation (C5), regions/islands (Eq. 16 generalised), grid (C6),
             gates (C10), island terms D..H (Eqs. 17-21, C7), eta assembly (Eqs. 11, 15, C2),
             the 3-D form over the COI band (NEXT-3 / R10)

Parity status: every function is pinned by a `-m "not gpu"` test in tests/test_oracle_*.py
except where its docstring says "parity unpinned" (DESIGN.md lists those); tests/test_oracle_mutants.py
plants 28 plausible slips in these modules one at a time and checks that the pins catch each.
"""
