"""Seeded synthetic inputs shared by the tests, the bench and the oracle checks.

This package holds NO arithmetic of the decoding method (no check/variable-node
update, no syndrome test of a decoded word): it only builds the inputs the
paper's decoder consumes —

* stand-in MET-LDPC parity-check matrices shaped like the paper's Table 1
  (Table 1, lines 61-68; the real ensembles of ref. [WANGRA] are not
  published) -> :mod:`synth.codes`;
* Bob/Alice CV-QKD frames after 8-dimensional multidimensional reconciliation
  (PAPER.md lines 20-24): Bob's bits U, his syndrome S_B = H U^T (Step 1,
  PAPER.md line 121), Alice's rotated observation V -> :mod:`synth.frames`.

Both the CUDA path and ``oracle/`` read these inputs; neither is imported here.
"""
