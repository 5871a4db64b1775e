"""ELIS ISRTF oracle -- TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct CPU implementation (numpy, fp64) of what the
hot path computes, written from PAPER.md (/root/reference/PAPER.md, arXiv
2505.09142).  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import it.  The product path
(``paper_2505_09142_b200``) never imports it and shares no code with it; the
only shared module is the seeded input generator
``paper_2505_09142_b200/inputs.py`` which holds none of the method's arithmetic.

Modules
  encoder.py  BGE/BERT bidirectional encoder forward, per request
  head.py     pooling + eight-FC regression head
  select.py   ISRTF / FCFS key + batch selection with preemption flags
              (Alg. 1 lines 10-19)
  sim.py      window-level scheduling simulator used for the JCT pins
              (Alg. 1)

Parity status per function is listed in DESIGN.md "Oracle pins".  Predictor
*quality* against the paper's MAE 19.923 / R^2 0.852 is "parity
unpinned": it needs trained weights and data that are not available offline.
"""
