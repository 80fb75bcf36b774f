"""B200-native executor for TACCL-synthesized collective schedules (arXiv 2111.04867).

* `taccl` — ctypes binding of the C ABI in include/taccl.h (libtaccl.so, built in-tree).
* `generator` — offline CPU schedule generator (templates, greedy stand-in, lowering).
* `inputs` — seeded synthetic inputs shared by tests and bench (no method arithmetic).
"""
