"""bench.py helpers that need no GPU: the multi-GPU collective figures
(algbw / busbw of the sharded rounds' all-reduce and all-gather)."""

import os
import sys

import pytest

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def test_collective_bw_busbw_factors():
    meta = {"allreduce_bytes": 4 << 30, "allgather_bytes": 1 << 30}
    kern = {"nccl_allreduce_min": 10.0, "nccl_allgather": 2.0, "nccl_allgather_changes": 0.5}
    c = bench.collective_bw(meta, kern, 8)
    ar, ag = c["allreduce_min"], c["allgather"]
    assert ar["algbw_gbs"] == pytest.approx((4 << 30) / 10e-3 / 1e9, rel=1e-3)
    assert ar["busbw_gbs"] == pytest.approx(ar["algbw_gbs"] * 2 * 7 / 8, rel=1e-3)
    assert ag["ms_per_step"] == pytest.approx(2.5)
    assert ag["busbw_gbs"] == pytest.approx(ag["algbw_gbs"] * 7 / 8, rel=1e-3)


def test_collective_bw_without_collectives():
    c = bench.collective_bw({}, {}, 2)
    assert c["allreduce_min"]["algbw_gbs"] is None and c["allgather"]["busbw_gbs"] is None
