"""ORACLE — TEST INFRASTRUCTURE ONLY.

CPU restatement of the reference's (arXiv 2203.06638 ``asyncsgd``) algorithm
for the LPP-SGD hot path, used as the *checker* of the CUDA product path.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import or execute anything
under ``oracle/``.  The product package ``paper_2203_06638_b200`` never
imports it and has no CPU fallback.

Parity pinning: every restatement here is checked against golden vectors
generated from the reference itself (``tests/golden/make_golden.py`` imports
a scratch build of ``/root/reference/pkg``) — see tests/test_oracle_golden.py.

Modules
  data.py        make_blobs restatement            (ref data.py:34-52)
  mlp.py         MlpObjective restatement (fp64)   (ref objectives.py:200-319)
  schedule.py    serialized canonical schedule     (ref engine.py:315-453)
  apply_ref.c    fp32 restatement of the kernels' per-element arithmetic
                 (ref _atomics.c:58-74, 186-215, 312-344; engine.py:199-229,418-421)
  native.py      ctypes loader for apply_ref.c and the reference-compiled
                 oracle/_ref/_atomics*.so
  engine_port.py threaded CPU engine port (ref engine.py:289-523) for the
                 CPU baseline arm
"""
