"""ORACLE -- test infrastructure, not product code.

CPU restatements of the reference algorithm on the MG-WFBP data path, used only
as the checker by ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py``.  Nothing in
``paper_1811_11141_b200`` imports this package.

Parity pinned: ``tests/test_oracle.py`` checks these restatements against golden
vectors produced by running the unmodified reference
(``/root/reference/pkg/src/mgwfbp``) -- its real multi-process TCP ring -- via
``tests/golden/make_golden.py``.
"""
