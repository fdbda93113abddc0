"""fp64 CPU ORACLE for the Gauss-Newton H·v hot path — TEST INFRASTRUCTURE ONLY.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s cpu_baseline / `--impl reference`
legs may import, call or execute anything under `oracle/`. The product path
(`paper_2507_10804_b200/`) never imports it and must fail loudly when its CUDA library is
missing; the two share no code (no kernels, headers, helpers, constant generators, pre- or
post-processing). Only the seeded input generators in `workloads/` (pure data, no method
arithmetic) serve both.

Contents
- `oracle.wave`  : the discrete acoustic forward map, Born (J), adjoint + imaging (J^T),
                   gradient and Gauss-Newton H·v, with FULL / CHECKPOINT / BOUNDARY storage
                   of the forward history.
- `oracle.psido` : the low-rank-symbol pseudo-differential operator apply, its adjoint and
                   symmetric variant (Eq. equ:lr-psido).

Pinning: every function is checked by `tests/test_oracle_*.py` (marker
"not gpu") against closed forms, invariants, brute force and special cases, never against
itself. Functions with no such pin are listed as "parity unpinned" below.

Parity unpinned: the absolute amplitude conventions of the wave path (1/h^2 point-source
scale, Euclidean inner products, sigma = 1 noise, Ricker delay t0 = 1/f; SURVEY.md §8(c)
C7, C9, C11, C12) have no external reference value — the paper prints no trace, gradient or
H·v numbers ("proprietary"). The pins fix the operators' internal
consistency and physics (adjoint identity, symmetry, finite differences, reciprocity,
travel time, Green's function), not those conventions.
"""
