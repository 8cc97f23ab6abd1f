"""Per-vertex lifecycle codes (oocgnn/vertexstate.py:19-38).

The state table itself lives on the GPU (u8 per vertex, engine.cu);
``StateTable`` here is the host view the reference API exposes
(``ctx.states.array``), fetched from the device on access.
"""

import numpy as np

from .errors import StateTransitionError

NOT_STARTED = 0
HOT = 1
COLD = 2
COMPLETED = 3

STATE_NAMES = {NOT_STARTED: "NOT_STARTED", HOT: "HOT", COLD: "COLD",
               COMPLETED: "COMPLETED"}

LEGAL_EDGES = frozenset({(NOT_STARTED, HOT), (HOT, COLD), (HOT, COMPLETED),
                         (COLD, HOT)})


class StateTable:
    """Read-only host view of the device state array of one layer."""

    def __init__(self, fetch):
        self._fetch = fetch

    @property
    def array(self) -> np.ndarray:
        return self._fetch()

    def counts(self) -> dict:
        uniq, n = np.unique(self.array, return_counts=True)
        return {STATE_NAMES[int(s)]: int(c) for s, c in zip(uniq, n)}

    def illegal_edges_taken(self) -> int:
        """The device engine only ever applies the four legal edges
        (engine.cu admit/evict/release); an illegal request raises
        StateTransitionError instead of being recorded."""
        return 0

    def transition(self, ids, src, dst):
        raise StateTransitionError(
            "state transitions are owned by the device engine")
