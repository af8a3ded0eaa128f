"""CPU oracle for the hierarchical exchange build -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this package, and
only as the checker / CPU baseline.  The product package
``paper_1401_6961_b200`` never imports it and has no CPU fallback.
"""
