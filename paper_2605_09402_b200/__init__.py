"""B200-native broadcast layer-wise GNN inference (ATLAS hot path).

Drop-in for the layer-wise inference API of the reference ``oocgnn``
package: model/layer definitions and formats (``storage``), the per-layer
operator triple (``orchestrator``), the transform backends (``compute``)
and the pipeline entry points (``runtime``). All compute runs in the
sm_100a library ``libatlas_b200.so`` through its C-ABI
(include/atlas_b200.h); there is no CPU fallback.
"""

__version__ = "0.1.0"

from .storage import (  # noqa: F401
    GraphCSR,
    LayerWeights,
    ModelKind,
    ModelWeights,
    generate_synthetic,
    random_weights,
    read_csr,
    read_weights,
    write_weights,
)
