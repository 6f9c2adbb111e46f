"""TEST INFRASTRUCTURE ONLY — the CPU oracle for the LINKS hot path.

This package is a numpy restatement of the reference ``linkatlas`` algorithms
on the data-parallel path (solver / curves / atlas scan).  It exists to CHECK
the CUDA product path, never to stand in for it:

* only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
  ``cpu_baseline`` / ``--impl reference`` legs may import it;
* the product package ``paper_2208_14567_b200`` must never import it.

Parity pin: the restatement is checked against golden vectors produced by the
reference itself (``tests/golden/make_golden.py`` imports ``/root/reference``
in the build container and writes ``tests/golden/*.npz``); see
``tests/test_oracle_golden.py``.
"""
