"""B200-native GACE selectivity probe (arxiv 2512.19750 Measurement Engine).

The product is libgace.so (C-ABI in include/gace.h, kernels in csrc/); this
package is its thin Python binding.  It never imports oracle/."""
from .gace import (GaceError, Table, table_attach, table_attach_host, derive, gate,  # noqa: F401
                   kernel_launches, PRED_DTYPE, PAIR_DTYPE, DistInfo)
