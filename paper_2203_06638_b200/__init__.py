"""B200-native LPP-SGD data-parallel hot path (arXiv 2203.06638).

Drop-in for the reference ``asyncsgd`` trainer/optimizer API on the hot
path: ``RunConfig`` / ``run_experiment`` / ``RunResult``,
``ParamStore`` / ``AtomicCounter``, ``select_block`` / ``balanced_boundaries``,
``lr_at`` / ``sync_every``.  The arithmetic runs in the C-ABI CUDA library
``lib/liblpp_b200.so`` (sources in ``csrc/``, ABI in ``include/lpp_b200.h``);
modules that touch device memory import it eagerly and fail loudly if it
has not been built — there is no CPU fallback.

Pure host-side schedule logic (partition, schedules) imports without the
library so it can be unit-tested on CPU.
"""

__version__ = "0.1.0"
