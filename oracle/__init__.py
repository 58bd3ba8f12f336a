"""CPU oracle for the Hessian-block / LMP-PCG hot path.

TEST INFRASTRUCTURE ONLY.  Nothing in ``paper_2605_23571_b200`` imports this
package; only ``tests/``, ``__graft_entry__.smoke()`` and the ``cpu_baseline`` /
``--impl reference`` legs of ``bench.py`` may use it, and only as the checker
or the timed CPU baseline -- never as the product path.

This is a plain numpy restatement of the reference algorithm
(``/root/reference/pkg/src/edasketch``), one module per reference module,
each function citing the reference ``file:line`` it follows.  Floating-point
operations are written in the same evaluation order as the reference so that
the restatement reproduces it bit for bit on the LAPACK-free paths (model,
observation operator, FFT covariance factor, Hessian apply, rhs, cost, PCG
without a preconditioner).  The LAPACK stages (QR/Cholesky/SVD in
``nystrom``) call the same numpy/scipy routines as the reference.

Parity pin: ``tests/golden/make_golden.py`` imports the real reference in the
build container and writes ``tests/golden/*.npz``; the CPU tests
(``tests/test_oracle_pins.py``) require this restatement to match those
vectors (bit-exact where noted) and the reference's own harness fixtures
(``pkg/frontend/test/fixtures/*.csv``, extracted to ``tests/golden``).
"""
