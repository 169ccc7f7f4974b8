"""CPU oracle for the syndrome BP decoder of arXiv 1711.01783 -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this package.  The
product path (``paper_1711_01783_b200``) never does, and shares no code with it.

* :mod:`oracle.bp`      -- ctypes wrapper of ``bp_oracle.c``: M2 (fp64 plain
  definition) and M3 (fp32 replay of the kernel precision), PAPER.md Steps 1-5.
* :mod:`oracle.literal` -- M1: Eqs. (1)-(5) literally, ratio domain, fp64, no
  degree-1 skip; tiny codes only.
* :mod:`oracle.brute`   -- exhaustive coset enumeration: bitwise MAP and block
  ML (ground truth for tiny codes).
"""
