"""CPU oracle for the QTT hot path — TEST INFRASTRUCTURE ONLY.

This package is a numpy restatement of the reference algorithms in
``qttfem`` (arXiv 2501.07778, mounted read-only at /root/reference during
development).  It is the *checker*: only ``tests/``, ``__graft_entry__.smoke``
and ``bench.py``'s CPU-baseline / ``--impl reference`` legs may import it.
The product package ``paper_2501_07778_b200`` never imports anything from
here and has no CPU fallback.

Pinning: every function is checked against golden vectors produced by the
reference itself (``tests/golden/make_golden.py`` imports the reference in
the development container and writes ``tests/golden/*.npz``), see
``tests/test_oracle_golden.py``.  Parity is therefore *pinned*.
"""
