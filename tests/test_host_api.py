"""Host-side behaviour of the drop-in API that needs no GPU: argument checks
and error classes (mirroring the reference's tests/test_analytics.py:38-44,
tests/test_traffic.py:71-77,157-159,194-206), partition rules
(tests/test_partitioning.py, tests/test_acceptance.py:148-194) and schedulers."""

import numpy as np
import pytest

import paper_2510_14050_b200 as nm
from paper_2510_14050_b200 import partitioning as pt


def test_reduction_argument_errors_precede_device_work():
    g = nm.make_inline_scheduler()
    with pytest.raises(ValueError):
        nm.sum_reduce([1], g, batch_count=0)
    with pytest.raises(TypeError):
        nm.sum_reduce(np.array([1.5, 2.5]), g)
    with pytest.raises(ValueError):
        nm.max_scan([1], g, batch_count=0)


def test_malformed_csr_rejected_before_device_work():
    with pytest.raises(nm.MatrixFormatError):
        nm.to_flat(nm.TrafficMatrix(0, 2, [0, 2], [0, 1], [1, 1]))
    with pytest.raises(nm.MatrixFormatError):
        nm.to_flat(nm.TrafficMatrix(0, 2, [0, 1, 2], [0, 1], [1, 0]))
    with pytest.raises(nm.MatrixFormatError):
        nm.to_flat(nm.TrafficMatrix(0, 2, [0, 2, 2], [1, 0], [1, 1]))
    with pytest.raises(nm.MatrixFormatError):
        nm.to_flat(nm.TrafficMatrix(0, 2, [0, 2, 2], [1, 1], [1, 1]))
    nm.TrafficMatrix(0, 3, [0, 1, 1, 3], [2, 0, 1], [1, 1, 1]).validate()  # decrease at a row start is legal
    assert issubclass(nm.MatrixFormatError, ValueError)


def test_stream_and_build_argument_errors():
    with pytest.raises(ValueError):
        nm.PacketStream(np.array([0, 1]), np.array([0]), np.ones(2, bool), 4)
    with pytest.raises(ValueError):
        nm.PacketStream(np.array([0, 5]), np.array([0, 1]), np.ones(2, bool), 4)
    with pytest.raises(ValueError):
        nm.build_matrices(nm.generate_packets(4, 4, seed=0), 0)
    assert nm.build_matrices(nm.generate_packets(0, 4, seed=1), 8) == []
    with pytest.raises(ValueError):
        nm.matrix_from_pairs([0], [0], 0)
    with pytest.raises(ValueError):
        nm.matrix_from_pairs([0], [0], 2**31 + 1)
    with pytest.raises(ValueError):
        nm.generate_packets(-1, 4, seed=0)


def test_generate_packets_matches_reference_restatement():
    from oracle import netmeter_oracle as orc

    s = nm.generate_packets(5000, 77, seed=42, invalid_fraction=0.2)
    rs, rd, rv = orc.generate_packets(5000, 77, 42, 0.2)
    assert np.array_equal(s.src, rs) and np.array_equal(s.dst, rd) and np.array_equal(s.valid, rv)
    # anonymize runs on the GPU: tests/test_gpu_anonymize.py


def test_partition_rules_exhaustive_small():
    for parts in range(1, 17):
        for total in range(0, 600):
            spans = pt.partition_even(total, parts).spans
            at = 0
            lens = []
            for off, ln in spans:
                assert off == at
                at += ln
                lens.append(ln)
            assert at == total and max(lens) - min(lens) <= 1
            assert lens == sorted(lens, reverse=True)
    plan = pt.partition_even(10, 3)
    assert pt.batch_table(plan, 2) == [[(0, 2), (4, 2), (7, 2)], [(2, 2), (6, 1), (9, 1)]]
    assert [b.view for b in pt.make_batches(plan, 2)] == [(0, 2), (2, 2), (4, 2), (6, 1), (7, 2), (9, 1)]
    with pytest.raises(ValueError):
        pt.partition_even(5, 0)
    with pytest.raises(ValueError):
        pt.make_batches(plan, 0)


def test_device_group_scheduler_contract():
    with nm.make_group_scheduler([2, 2, 2, 2]) as g:
        assert g.resource_count == 4
        seen = [None] * 10
        g.run_bulk(10, lambda i, r, out: out.__setitem__(i, r), (seen,))
        assert seen == [0, 0, 0, 1, 1, 1, 2, 2, 3, 3]
    assert nm.make_group_scheduler(3).resource_count == 3
    with pytest.raises(ValueError):
        nm.make_group_scheduler(0)
    with pytest.raises(ValueError):
        nm.make_group_scheduler([1, 1], workers_per_resource=2)
    assert nm.make_inline_scheduler().resource_count == 1


def test_report_serialisation_order():
    r = nm.AggregateReport(6, 3, 2, 2, 2, 2)
    assert list(r.to_dict()) == ["valid_packets", "unique_links", "unique_sources", "max_fanout",
                                 "unique_destinations", "max_fanin"]
    assert nm.AggregateReport.from_dict(r.to_dict()) == r
    s = nm.Stats9(6, 3, 3, 2, 3, 2, 2, 4, 2)
    assert s.report() == r and s.astuple() == (6, 3, 3, 2, 3, 2, 2, 4, 2)


def test_group_run_bulk_every_index_once_concurrently():
    """run_bulk (senders.py:32-38 contract): each index once, contiguous partition_even
    spans per resource (resources.py:107-113), the resources' spans concurrent."""
    import threading

    seen = []
    lock = threading.Lock()
    meet = threading.Barrier(4, timeout=10)  # only passable if the 4 spans run at once
    spans = nm.partition_even(10, 4).spans

    def task(i, rid, scale):
        with lock:
            seen.append((i, rid, scale))
        if i == spans[rid][0]:
            meet.wait()

    with nm.make_group_scheduler(4) as g:
        g.run_bulk(10, task, (3,))
    assert sorted(i for i, _, _ in seen) == list(range(10))
    for i, rid, scale in seen:
        off, ln = spans[rid]
        assert off <= i < off + ln and scale == 3

    def boom(i, rid):
        if i == 7:
            raise RuntimeError("task failed")

    with pytest.raises(RuntimeError, match="task failed"):
        nm.make_group_scheduler(3).run_bulk(9, boom, ())
    with pytest.raises(ValueError):
        nm.make_group_scheduler([1, 0])
