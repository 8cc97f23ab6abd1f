"""Dense layer transform and its backend registry (oocgnn/compute.py).

Backends keep the reference's plug-in shape (``name``, ``max_batch_rows``,
``apply(batch, weight, bias)``, ``register_backend``/``get_backend``):

* ``stable`` (default, like the reference) runs the SIMT kernel of
  csrc/transform.cu that evaluates the reference's fixed k-order f32 chain
  per element: outputs are bit-identical to oocgnn's MatmulBackend.
* ``tcgen05`` runs the tensor-core kernel (csrc/transform_tc.cu): 3xTF32
  split products on tcgen05.mma with TMEM accumulators; fp32-level
  accuracy, not bit-identical. ``blas`` is an alias (the reference's
  "fast but batch-shape dependent" slot).

A user backend without a device ``code`` is honoured as a host plug-in
(its ``apply`` runs on numpy arrays), exactly as the reference does.
"""

import numpy as np

from . import _native as N
from .errors import ConfigError


class MatmulBackend:
    name = "stable"
    max_batch_rows = None
    code = N.BACKEND_STABLE

    def apply(self, batch: np.ndarray, weight: np.ndarray,
              bias: np.ndarray) -> np.ndarray:
        return _apply_device(self.code, batch, weight, bias, relu=False)


class Tcgen05Backend(MatmulBackend):
    name = "tcgen05"
    code = N.BACKEND_TCGEN05


class BlasBackend(Tcgen05Backend):
    name = "blas"


_BACKENDS = {"stable": MatmulBackend, "tcgen05": Tcgen05Backend,
             "blas": BlasBackend}


def register_backend(cls) -> None:
    _BACKENDS[cls.name] = cls


def get_backend(name):
    if isinstance(name, MatmulBackend) or hasattr(name, "apply"):
        return name
    try:
        return _BACKENDS[name or "stable"]()
    except KeyError:
        raise ConfigError(f"unknown compute backend {name!r}") from None


def device_code(backend):
    """Device backend code, or None for a host plug-in."""
    return getattr(backend, "code", None)


def _apply_device(code, batch, weight, bias, relu):
    import torch

    from .engine import transform_device

    x = torch.as_tensor(np.ascontiguousarray(batch, dtype=np.float32)).cuda()
    w = torch.as_tensor(np.ascontiguousarray(weight, dtype=np.float32)).cuda()
    b = torch.as_tensor(np.ascontiguousarray(bias, dtype=np.float32)).cuda()
    y = torch.empty((x.shape[0], w.shape[0]), dtype=torch.float32,
                    device="cuda")
    if x.shape[0]:
        transform_device(x.data_ptr(), x.shape[0], x.shape[1], x.stride(0),
                         w, b, relu, y, code)
    return y.cpu().numpy()


def transform(batch: np.ndarray, layer, *, apply_activation: bool,
              backend=None) -> np.ndarray:
    """out = act(batch @ W.T + bias) (oocgnn/compute.py:76-97)."""
    backend = get_backend(backend)
    if batch.shape[1] != layer.in_dim:
        raise ConfigError(
            f"batch width {batch.shape[1]} != layer in_dim {layer.in_dim}")
    code = device_code(backend)
    if code is not None:
        return _apply_device(code, batch, layer.weight, layer.bias,
                             apply_activation)
    cap = backend.max_batch_rows
    if cap and len(batch) > cap:
        out = np.concatenate([backend.apply(batch[i:i + cap], layer.weight,
                                            layer.bias)
                              for i in range(0, len(batch), cap)])
    else:
        out = backend.apply(batch, layer.weight, layer.bias)
    out = np.asarray(out, dtype=np.float32)
    if apply_activation:
        np.maximum(out, 0.0, out=out)
    return out


class GraduationSink:
    """Collects graduated (ids, rows) batches in arrival order; the
    operator path hands it what ``process_chunk`` graduates
    (oocgnn/compute.py:125-170 minus the thread hand-off, which the GPU
    pipeline does not need)."""

    def __init__(self, capacity_bytes: int = 0, dim: int = 0, *_):
        self.ids = []
        self.rows = []
        self.rows_shipped = 0

    def add_batch(self, ids, rows) -> None:
        self.ids.append(np.asarray(ids))
        self.rows.append(np.asarray(rows))
        self.rows_shipped += len(ids)

    def finish(self) -> None:
        pass
