"""TEST INFRASTRUCTURE ONLY — the CPU oracle for the FIDS per-time-step path.

Nothing in the product package (`paper_2002_11978_b200`) may import this
package.  Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s CPU
baseline / `--impl reference` arm use it, and only as the checker or the
timed CPU reference, never as the thing measured on the GPU.

Parity pin: `oracle/gen_golden.py` imports the upstream reference
(`/root/reference/pkg/src/tsfrac`, available only in the build container),
runs it on seeded inputs and writes `tests/golden/*.npz`;
`tests/test_oracle_golden.py` checks this restatement against those vectors.
"""

from .tsfrac_oracle import *  # noqa: F401,F403
