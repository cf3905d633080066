"""hiccl-b200: B200-native HiCCL collective execution path.

Host C++ composer/factorizer/pipeliner + persistent sm_100a executor behind
a C ABI (include/hiccl.h). ``paper_2408_05962_b200.hiccl`` is the Python face
of that ABI; importing it loads lib/libhiccl.so and fails if it was not built
(``python -m paper_2408_05962_b200.build``).
"""
