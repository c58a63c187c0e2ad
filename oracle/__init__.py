"""TEST INFRASTRUCTURE ONLY — the CPU oracle for the MSDA hot path.

This package restates, on the CPU, the reference algorithm of
``mvtrack3d.features`` (``/root/reference/pkg/src/mvtrack3d/features.py``)
and the OAE / projection helpers that feed it.  It exists so that the
``tests/`` suite, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` leg can check and time the GPU
product against an independent implementation.

Nothing in ``paper_2601_10819_b200`` (the product) may import this package;
``tests/test_product_isolation.py`` enforces that.

Parity pinning: the restatement is checked against golden vectors generated
by importing the real reference (``tests/golden/make_golden.py``), see
``tests/test_oracle_golden.py``.
"""
