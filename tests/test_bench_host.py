"""Host logic of bench.py: the N > 1 reduction (max over ranks, world_size 2 on gloo), the
whole-job value, the clocks summary and the roofline object."""
import os
import socket

import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

import bench  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    dist.init_process_group("gloo", init_method="tcp://127.0.0.1:%d" % port, rank=rank, world_size=world)
    try:
        ms = 10.0 + 5.0 * rank
        m = bench.max_over_ranks(ms, "cpu")
        bench.barrier("cpu")
        out[rank] = (m, bench.whole_job_value(1 << 20, world, m))
    finally:
        dist.destroy_process_group()


def test_max_over_ranks_gloo_world2():
    port = _free_port()
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
        res = dict(out)
    assert res[0][0] == res[1][0] == 15.0
    assert res[0][1] == pytest.approx(2 * (1 << 20) / 15e-3)


def test_single_process_identity():
    assert bench.max_over_ranks(3.5) == 3.5
    assert bench.whole_job_value(1000, 1, 2.0) == pytest.approx(5e5)


def test_clock_summary_flags_throttle():
    rows = [dict(sm=1965.0, max=1965.0, hw_slowdown="Not Active", hw_thermal_slowdown="Not Active",
                 sw_thermal_slowdown="Not Active", sw_power_cap="Active"),
            dict(sm=1900.0, max=1965.0, hw_slowdown="Active", hw_thermal_slowdown="Not Active",
                 sw_thermal_slowdown="Not Active", sw_power_cap="Not Active")]
    c = bench.summarize_clocks(rows)
    assert c["sm_mhz"] == pytest.approx(1932.5) and c["sm_max_mhz"] == 1965.0
    assert c["reasons"] == ["hw_slowdown", "sw_power_cap"]
    assert bench.summarize_clocks([])["reasons"] == ["no samples"]


def test_roofline_entry_overlap_span():
    stats = {"p2p_pairs": 1000, "m2l_entries": 4000}
    inputs = {"fp64_tflops_measured": 34.0,
              "kernels": {"m2l": {"fp64_flops_per_entry": 100.0, "dram_bytes_per_launch": 123},
                          "p2p": {"fp64_flops_per_entry": 50.0, "dram_bytes_per_launch": 7}}}
    r = bench.roofline_entry({"near": 1.0, "m2l": 4.0, "overlap_span": 5.0}, 2, stats, inputs)
    assert r["bound"] == "alu" and r["unit"] == "TFLOP/s" and r["span_ms"] == 2.5
    assert r["achieved"] == pytest.approx((4000 * 100.0 + 1000 * 50.0) / 2.5e-3 / 1e12)
    assert r["frac"] == pytest.approx(r["achieved"] / 34.0) and r["traffic"] == 130
    assert r["kernels"]["m2l"]["launch_ms_concurrent"] == 2.0


def test_roofline_entry_stored_m2l():
    """Stored M2L blocks: the dominant kernel is the HBM stream; achieved = algorithmic bytes
    (16 B per entry + 20 B per source-stream element + 16 B per output) / its launch time."""
    stats = {"p2p_pairs": 1000, "m2l_entries": 4000, "m2l_stored_entries": 4000, "m2l_stored": 1, "m2l_stream_len": 100, "n_loc": 50,
             "operator_bytes": 10000, "n": 64}
    inputs = {"fp64_tflops_measured": 34.0,
              "kernels": {"m2l_stored": {"dram_bytes_per_launch": 70000, "ncu_time_ms": 0.5},
                          "p2p": {"fp64_flops_per_entry": 50.0, "dram_bytes_per_launch": 7}}}
    r = bench.roofline_entry({"near": 2.0, "m2l": 1.0, "overlap_span": 3.0}, 2, stats, inputs, ms_per_step=2.0)
    nbytes = 16 * 4000 + 20 * 100 + 16 * 50
    assert r["bound"] == "hbm" and r["unit"] == "GB/s"
    assert r["algorithmic_bytes_per_launch"] == nbytes
    assert r["achieved"] == pytest.approx(nbytes / 0.5e-3 / 1e9)
    assert r["frac"] == pytest.approx(r["achieved"] / r["peak"]) and r["traffic"] == 70000
    assert r["concurrent"]["p2p"]["achieved"] == pytest.approx(1000 * 50.0 / 1e-3 / 1e12)
    st = r["step"]
    assert st["bound_ms"] == max(st["alu_ms"], st["hbm_ms"]) and st["frac"] == pytest.approx(st["bound_ms"] / 2.0)
