"""CPU FP64 oracle for the KFBI interface-problem apply and BIE solve (arXiv 2404.15249).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and bench.py's
``cpu_baseline`` / ``--impl reference`` legs may import or execute anything here.  The
product path (``paper_2404_15249_b200``) never imports it and shares no code, tables or
constants with it; the two meet only through the seeded inputs of ``workloads``.

Plain, slow, obviously correct: NumPy/SciPy FP64, vectorised only where a formula is
applied elementwise; each function cites the PAPER.md passage (``P:<line>``) it follows.
Where the paper is silent or garbled the reading of SURVEY.md §8(c) / DESIGN.md is used
and named (R<n>).

Parity status: every function is pinned by ``tests/test_oracle_*.py`` against closed
forms, brute force or worked examples.  No function is
"parity unpinned", except where a module header says otherwise.
"""
