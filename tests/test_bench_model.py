"""bench.py's per-kernel algorithmic byte model
reads the path a build took from dmst_stats; check it follows the path
fields (no GPU needed: a stand-in stats object)."""
from __future__ import annotations

import bench


class _Stats:
    def __init__(self, v0_chase):
        # views 0..3 of a random 1M-edge tree: (n_alpha, n_leaf, n_chain, n_k)
        self._counts = [(262_000, 262_000, 476_000, 1_000_000), (65_000, 66_000, 131_000, 262_000),
                        (16_000, 17_000, 32_000, 65_000), (0, 4_000, 12_000, 16_000)]
        self.num_levels = 3
        self.view_vertices = [1_000_001, 262_000, 65_000, 16_000]
        self.sort1_passes = 2
        self.sort2_passes = 3
        self._info = {"mi_bucketed_views": [0, 1], "mi_direct_views": [2, 3], "sort1_narrow": True,
                      "sort1_local": None, "v0_chase": v0_chase}

    def view_kind_counts(self):
        return self._counts

    def path_info(self):
        return self._info


def test_chased_view0_moves_bytes_from_v2_to_select():
    plain = bench.kernel_bytes(_Stats(None), 1_000_000, 1_000_001)
    chased = bench.kernel_bytes(_Stats("chase"), 1_000_000, 1_000_001)
    # V2 no longer runs on view 0: its 12 B per view-0 vertex are gone
    assert plain["v2"] - chased["v2"] == 12.0 * 1_000_001
    # the select reads 8-B maxIncident entries instead of 4-B vertex-map entries
    # for every endpoint it needs (first end of chain edges, both ends of alpha edges)
    assert chased["select_edges"] - plain["select_edges"] == 4.0 * (476_000 + 2 * 262_000)
    for k in plain:
        if k not in ("v2", "select_edges"):
            assert plain[k] == chased[k]


def test_byte_model_counts_view0_chain_gathers():
    b = bench.kernel_bytes(_Stats(None), 1_000_000, 1_000_001)
    views_n = [1_000_000, 262_000, 65_000]
    alpha = 262_000 + 65_000 + 16_000
    assert b["select_edges"] == 9.0 * sum(views_n) + 4.0 * 1_000_000 + 20.0 * alpha + 4.0 * 476_000 + 16.0 * (65_000 + 16_000)
