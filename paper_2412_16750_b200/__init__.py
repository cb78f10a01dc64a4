"""B200-native differentiable IDM hot path (arXiv 2412.16750).

The CUDA path lives behind the C-ABI library ``libidm.so`` (``include/idm.h``); the Python
binding is :mod:`paper_2412_16750_b200.idm`.  Import it explicitly; this package init stays
light so the seeded generator (:mod:`paper_2412_16750_b200.synth`) can be used on CPU-only hosts.
"""
