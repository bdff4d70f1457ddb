"""B200-native QTT tensor-train hot path (drop-in for ``qttfem``, arXiv 2501.07778).

Modules mirror the reference package: ``ttcore`` (TT algebra), ``indexing``
(Z-order maps), ``element``/``assembly`` (QTT stiffness/load assembly),
``coupling`` (global system, Dirichlet), ``solver`` (AMEn solve), plus the
host-side geometry ``mesh``/``material``/``topology``.  All arithmetic runs
in ``lib/libqttb200.so`` (hand-written sm_100a kernels, C ABI in
``include/qtt_b200.h``); there is no CPU fallback.
"""

__version__ = "0.1.0"
