"""ORACLE -- TEST INFRASTRUCTURE ONLY.

CPU restatement (``core.py`` + ``lines.c``) of the reference algorithm for the
SLDG / spline hot path, plus an optional build of the reference's own
compiled line kernels (``_ref/``).  Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s CPU legs may use this package; the product package
``paper_1803_02143_b200`` never imports it.
"""
