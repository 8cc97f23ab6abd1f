"""Float64 gather oracle (TEST INFRASTRUCTURE ONLY).

Restates ``oracle_inference`` (oocgnn/oracle.py:18-55): a scipy CSR
(dst, src) matrix product per layer in float64, mean = sum * 1/max(1,d_in),
SAGE concat [mean || self], GIN sum + (1+eps) self, ReLU on every layer
but the last. ``per_layer`` returns every layer's post-activation output
(the reference returns only the last).

Pinned: tests/test_cpu_boundary.py::test_gather_oracle_pinned_to_reference_oracle
checks the last layer, rounded to f32, equals the reference's
``oracle_inference`` output stored by make_golden for every golden case
(bit-exact); the cfg2-scale golden adds the reference's per-layer outputs
on sampled rows."""

import numpy as np
import scipy.sparse as sp

GCN, SAGE, GIN = 0, 1, 2


def gather_matrix(num_vertices, offsets, neighbors):
    src = np.repeat(np.arange(num_vertices, dtype=np.int64), np.diff(offsets))
    data = np.ones(len(src), dtype=np.float64)
    return sp.csr_matrix((data, (np.asarray(neighbors, np.int64), src)),
                         shape=(num_vertices, num_vertices))


def per_layer(num_vertices, offsets, neighbors, in_degrees, features, model,
              layers, gin_epsilon=0.0):
    """layers: list of (weight (out,in) f32, bias f32). Returns list of f64
    layer outputs."""
    adj = gather_matrix(num_vertices, offsets, neighbors)
    inv = 1.0 / np.maximum(np.asarray(in_degrees), 1).astype(np.float64)
    h = np.asarray(features, dtype=np.float64)
    outs = []
    for i, (w, b) in enumerate(layers):
        agg = adj @ h
        if model == GCN:
            x = agg * inv[:, None]
        elif model == SAGE:
            x = np.concatenate([agg * inv[:, None], h], axis=1)
        else:
            x = agg + (1.0 + gin_epsilon) * h
        h = x @ np.asarray(w, np.float64).T + np.asarray(b, np.float64)
        if i != len(layers) - 1:
            np.maximum(h, 0.0, out=h)
        outs.append(h)
    return outs
