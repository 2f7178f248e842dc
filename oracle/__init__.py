"""CPU oracle for the L3 codec — TEST INFRASTRUCTURE ONLY.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` legs may import this package. The product package
(``paper_2208_08711_b200``) never imports it and shares no code with it.

* ``oracle/l3ref.c``   — the oracle proper (plain C, §4.2-§4.3)
* ``oracle/l3ref.py``  — ctypes binding
* ``oracle/pymodel.py`` — a second, pure-Python model (bit strings, tiny inputs
  only) used to pin the C oracle's bit packing on brute-force cases.

Parity unpinned: byte-compatibility with the authors' own
L3 files (magic, tie order, base rule and offset width are not printed in the
paper), and the Table 4 ratios of the real datasets.
"""
