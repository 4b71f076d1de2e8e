"""CPU oracle for the SPD-KFAC optimizer-step hot path.

TEST INFRASTRUCTURE ONLY.  Nothing in the product package
(`paper_2107_06533_b200/`) imports this package; only `tests/`,
`__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` / `--impl reference`
leg may use it, and only as the checker (or the timed CPU reference arm),
never as the thing measured on the GPU or shipped.

It is a float64 numpy/scipy restatement of the reference package `kfacsched`
(`/root/reference/pkg/src/kfacsched`), function by function, with the
reference file:line each one follows.  The reference delegates its
arithmetic to numpy BLAS (`x.T @ x`, `@`) and scipy LAPACK
(`lapack.dpotrf`, `solve_triangular`) -- numpy>=1.24 / scipy>=1.10
(`pkg/pyproject.toml:10-13`, no lockfile); this image pins numpy 2.3 and
scipy 1.18, the same libraries the reference's own 183 tests pass with.

Parity of the restatement is pinned by `tests/test_oracle.py` against
  * the reference's frozen golden fixture `tests/data/aggregated_step_w4.json`
    (copied verbatim as data into `tests/golden/`),
  * the reference's known-answer tests (`tests/test_linalg.py:43-239`),
  * golden vectors produced by importing the reference itself in the dev
    container (`tests/golden/make_golden.py` -> `tests/golden/*.json/npz`).
"""

from .linalg import (  # noqa: F401
    NotPositiveDefinite,
    factor,
    factor_A,
    factor_G,
    damped_inverse,
    precondition,
    pack_upper,
    unpack_upper,
    kron_vec_precondition,
    im2col_rows,
    conv_grad_rows,
)
from .emulator import (  # noqa: F401
    mlp_forward_backward,
    dkfac_step,
    kfac_step_centralized,
    layer_kfac_update,
    run_fixture,
)
