"""The reference's cluster model restated in paper_1910_00932_b200.scaling,
pinned against the reference's own sim.cpp (oracle/_ref), plus the CSV and
validation behaviour."""
import pytest

from paper_1910_00932_b200 import ValidationError
from paper_1910_00932_b200 import scaling as sc


@pytest.mark.parametrize("nodes", [1, 2, 4, 8])
@pytest.mark.parametrize("ring", [True, False])
def test_step_time_matches_reference(ref, nodes, ring):
    p = sc.b200_profile(nodes=nodes)
    got = sc.step_time(p, per_gpu_batch=64, ring=ring)
    want = ref.step_time(p.as_list(), sc.TSM8F_FLOPS, sc.TSM8F_PARAMS, sc.TSM8F_INPUT_BYTES, 64,
                         3.0, ring)
    assert (got.t_compute, got.t_io, got.t_comm, got.t_step) == pytest.approx(want, rel=1e-15)


def test_io_bound_profile_matches_reference(ref):
    p = sc.ClusterProfile(nodes=3, gpus_per_node=6, peak_flops_per_gpu=1.25e14,
                          utilization=0.4, disk_bandwidth_per_node=2e8, net_latency=2e-5,
                          net_bandwidth=1.2e10)
    got = sc.step_time(p, per_gpu_batch=8)
    want = ref.step_time(p.as_list(), sc.TSM8F_FLOPS, sc.TSM8F_PARAMS, sc.TSM8F_INPUT_BYTES, 8)
    assert (got.t_compute, got.t_io, got.t_comm, got.t_step) == pytest.approx(want, rel=1e-15)
    assert got.bottleneck == "io"


def test_observed_scalability_matches_reference(ref):
    t = [(1, 0.0252), (2, 0.0255), (4, 0.0257), (8, 0.0262)]
    assert sc.observed_scalability(t) == pytest.approx(ref.observed_scalability(t), rel=1e-15)
    with pytest.raises(ValidationError):
        sc.observed_scalability([(2, 1.0)])
    with pytest.raises(ValidationError):
        sc.observed_scalability([(1, 0.0)])


def test_profile_validation():
    with pytest.raises(ValidationError, match="utilization"):
        sc.step_time(sc.ClusterProfile(peak_flops_per_gpu=1, utilization=1.5,
                                       disk_bandwidth_per_node=1, net_bandwidth=1))


def test_overlap_never_slower_and_single_gpu_equal():
    for n in (1, 2, 4, 8):
        p = sc.b200_profile(nodes=n)
        a, b = sc.step_time(p), sc.step_time_overlapped(p)
        assert b.t_step <= a.t_step
        if n == 1:
            assert a.t_step == b.t_step


def test_timings_csv(tmp_path):
    f = tmp_path / "t.csv"
    f.write_text("nodes,wall_seconds\n1,0.025\n4,0.0257\n")
    assert sc.load_timings_csv(f) == [(1, 0.025), (4, 0.0257)]
    f.write_text("gpus,seconds\n1,1\n")
    with pytest.raises(ValidationError, match="header"):
        sc.load_timings_csv(f)
