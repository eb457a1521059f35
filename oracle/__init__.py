"""CPU oracle for the INT8 training hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package.  The product package
(``paper_1912_12607_b200``) never imports it: the CUDA path fails loudly
instead of falling back to anything here.

``oracle.lib``  -- ctypes bindings of ``liboracle.so`` (C restatement in
                   ``oracle.c``, each function citing reference file:line).
``oracle.ref``  -- ctypes bindings of ``_ref/libi8t_ref.so`` (the unmodified
                   reference compiled from /root/reference by the Makefile),
                   available only where it was built.
"""
