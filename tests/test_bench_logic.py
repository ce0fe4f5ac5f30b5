"""bench.py's measurement logic on a fake runtime (CPU): the knee search picks
the feasible rate with the most completed inferences/s (not the highest
feasible rate); a rate is feasible only when EVERY window of its run has HP
miss 0 and LP loss < 2 % (admission rejections count as lost); the timed run
is never re-measured at the same rate — any failing window steps the rate
down and repeats the whole run; windows with a GPU-wide pause are tagged and
exempt under the secondary, pause-excluded criterion."""

from types import SimpleNamespace

import bench
from paper_2504_08795_b200.runtime import window_ok


def _rep(jps, missed_hp=0, released_lp=1000, missed_lp=0, rejected_lp=0, accepted_lp=None):
    accepted_lp = released_lp - rejected_lp if accepted_lp is None else accepted_lp
    return SimpleNamespace(jps=jps, completed_hp=int(jps), completed_lp=1, missed_hp=missed_hp, missed_lp=missed_lp,
                           released_lp=released_lp, rejected_lp=rejected_lp, accepted_lp=accepted_lp,
                           dmr_lp=(missed_lp / accepted_lp) if accepted_lp else 0.0,
                           response_hp=SimpleNamespace(p99=0.0005))


def _win(imgs, missed_hp=0, released_lp=100, lost_lp=0, stalls=0):
    return {"released_hp": 100, "released_lp": released_lp, "missed_hp": missed_hp, "missed_lp": 0,
            "rejected_lp": lost_lp, "lp_loss": lost_lp / released_lp, "completed_images": imgs, "stalls": stalls}


class FakeRuntime:
    """Throughput rises with the rate up to a cliff at 1000/task where admission
    rejects every LP job, HP misses start at 1300. The first `pauses` runs at
    rates >= 600 have a 1.6 ms GPU-wide pause in window 3, which misses HP jobs
    there (periods below pause + response time); `poison` also makes every
    later window lose LP jobs (an MRET sample inflated by the pause keeping a
    task rejected — what the executor's pause-excluded samples prevent)."""

    def __init__(self, pauses=0, poison=False):
        self.rate = 0.0
        self.afet = {}
        self.runs = []
        self.pauses = pauses
        self.poison = poison

    def set_rate(self, r):
        self.rate = r

    def run(self, duration, warmup, full_load=None):
        r = self.rate
        self.runs.append(r)
        pause = len(self.runs) <= self.pauses and r >= 600

        def windows(warm, step, n):
            out = []
            for k in range(n):
                imgs = 8 * r * step if r < 1000 else 4 * r * step
                w = _win(imgs, missed_hp=3 if r >= 1300 else 0, lost_lp=100 if r >= 1000 else 0)
                if pause and k == 3:
                    w = _win(imgs, missed_hp=2, stalls=1)
                elif pause and k > 3 and self.poison:
                    w = _win(imgs, lost_lp=30)
                out.append(w)
            return out
        return SimpleNamespace(report=_rep(8 * r), windows=windows, stats={"stalls": 0}, trace=[],
                               stalls=[(warmup + 1.6, 0.0016)] if pause else [])


def test_lp_rejections_count_as_loss():
    assert bench.lp_loss(_rep(100, rejected_lp=30, missed_lp=0)) == 0.03
    assert not bench.feasible(_rep(100, rejected_lp=30))            # DMR 0 but 3 % of LP jobs lost
    assert bench.feasible(_rep(100, rejected_lp=10, missed_lp=5))   # 1.5 % lost
    assert not bench.feasible(_rep(100, missed_hp=1))
    assert window_ok(_win(10, lost_lp=1)) and not window_ok(_win(10, lost_lp=2))
    assert not window_ok(_win(10, missed_hp=1))


def test_knee_is_the_throughput_maximum_below_the_admission_cliff():
    rt = FakeRuntime()
    rate = bench.knee_search(rt, 400.0, 1.0, 0.5, lambda m: None)
    assert 900 < rate < 1000, rate


def test_timed_run_steps_down_until_every_window_passes():
    """Strict: a run with any failing window is not re-measured; after a run
    that failed only in a pause window the next rate's period covers the pause
    plus the p99 HP response (1 / (1.6 + 0.5 + 0.1) ms = 454.5/task)."""
    rt = FakeRuntime(pauses=100)      # every run at >= 600/task is hit by a pause
    args = SimpleNamespace(step_seconds=0.5, warmup=2, steps=20, timed_attempts=8)
    rate, res, s, clocks, wall, attempts = bench.timed_knee(rt, 950.0, args, lambda m: None, "t",
                                                            pause_floor=bench.pause_floor)
    assert [round(r, 2) for r in rt.runs] == [a["rate_per_task"] for a in attempts]   # one run per attempt
    assert len(attempts) == 2 and abs(rate - 1 / 0.0022) < 1e-6 and s["ok"] and s["windows_failed"] == 0
    assert attempts[0]["windows_failed"] == 1 and attempts[0]["windows_failed_without_pause"] == 0
    assert attempts[0]["longest_pause_ms"] == 1.6


def test_timed_run_without_pause_floor_steps_down_geometrically():
    rt = FakeRuntime(pauses=100, poison=True)
    args = SimpleNamespace(step_seconds=0.5, warmup=2, steps=20, timed_attempts=8)
    rate, res, s, clocks, wall, attempts = bench.timed_knee(rt, 950.0, args, lambda m: None, "t")
    assert rate < 600 and s["ok"]
    assert all(abs(r2 - 0.85 * r1) < 1e-9 for r1, r2 in zip(rt.runs, rt.runs[1:]))
    assert all(a["windows_failed"] == 17 and a["windows_failed_without_pause"] == 16 for a in attempts[:-1])


def test_pause_excluded_criterion():
    """ok_excl exempts the windows that saw a GPU-wide pause, nothing else."""
    rt = FakeRuntime(pauses=100)
    args = SimpleNamespace(step_seconds=0.5, warmup=2, steps=20, timed_attempts=8)
    rate, res, s, *_ = bench.timed_knee(rt, 950.0, args, lambda m: None, "t", criterion="ok_excl")
    assert rate == 950.0 and s["ok_excl"] and not s["ok"] and s["windows_with_pause"] == 1
    rt = FakeRuntime(pauses=100, poison=True)   # later windows failing without a pause still fail it
    rate, res, s, *_ = bench.timed_knee(rt, 950.0, args, lambda m: None, "t", criterion="ok_excl")
    assert rate < 600
    assert bench.knee_search(FakeRuntime(pauses=100), 400.0, 2.5, 0.5, lambda m: None, criterion="ok_excl") > 900


def test_summarize_counts_and_pause_attribution():
    ws = [_win(50), _win(50, missed_hp=1), _win(50, stalls=1, lost_lp=5), _win(50, lost_lp=5)]
    s = bench.summarize(ws, 0.5)
    assert s["windows_failed"] == 3 and s["windows_failed_without_pause"] == 2 and s["windows_with_pause"] == 1
    assert s["inf_per_s"] == 200 / 2.0 and s["missed_hp"] == 1 and not s["ok"] and not s["ok_excl"]


def test_reference_arm_prints_the_contract_line():
    """`bench.py --impl reference` (the reference's CPU path on the host) prints
    one JSON line with the contract keys, on CPU only."""
    import json
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    r = subprocess.run([sys.executable, str(root / "bench.py"), "--impl", "reference", "--steps", "1", "--warmup", "0",
                        "--cpu-seconds", "1"], capture_output=True, text=True, timeout=600, cwd=root)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "dtype", "config", "impl", "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0


def test_conv_algorithmic_bytes_resnet50():
    """The roofline's algorithmic bytes: every conv's weights + input + output
    (+ residual / fused branch input) once; ResNet-50 b1 convs sit below the
    B200 ridge point, so the roofline that bounds them is HBM."""
    import torch
    from paper_2504_08795_b200 import nets
    net = nets.build_network("resnet50", batch=1, n_stages=4, device=torch.device("cpu"))
    convs = [op for op in net.ops if op.kind == "conv"]
    nbytes = sum(bench.conv_algorithmic_bytes(op) for op in convs)
    wbytes = sum(op.layer.weight.numel() * 2 for op in convs)
    assert wbytes < nbytes < wbytes + 60e6
    assert sum(op.flops for op in convs) / nbytes < 1642e12 / 6547.8e9


def test_pause_excluded_knee_steps_up_while_passing():
    """step_up: after a passing continuous run the rate rises x1.08 (at most
    twice) while runs keep passing; the last passing run is reported."""
    rt = FakeRuntime()            # cliff at 1000/task
    args = SimpleNamespace(step_seconds=0.5, warmup=2, steps=20, timed_attempts=8)
    rate, res, s, *_ = bench.timed_knee(rt, 880.0, args, lambda m: None, "t", criterion="ok_excl", step_up=2)
    assert [round(r, 1) for r in rt.runs] == [880.0, 950.4, 1026.4]   # third run fails at the cliff
    assert abs(rate - 950.4) < 1e-6 and s["ok_excl"]
    rt = FakeRuntime()
    rate, *_ = bench.timed_knee(rt, 500.0, args, lambda m: None, "t", criterion="ok_excl", step_up=2)
    assert abs(rate - 500.0 * 1.08 ** 2) < 1e-6 and len(rt.runs) == 3


def test_overloaded_run_fails_every_window():
    """A run the executor stops as overloaded (buffer sets exhausted past the
    knee: runtime.BufferSetsExhausted) is an infeasible rate, not a crash: every
    window fails under both criteria, and the knee search steps below it."""
    from paper_2504_08795_b200.runtime import BufferSetsExhausted

    class Overloading(FakeRuntime):
        def run(self, duration, warmup, full_load=None):
            if self.rate >= 900:
                raise BufferSetsExhausted("daris_exec_run failed (13): buffer sets exhausted: 8 stage-0 launches")
            return super().run(duration, warmup, full_load)

    rt = Overloading()
    res, ws = bench.run_windows(rt, 0.1, 0.5, 4)
    assert len(ws) == 4 and all(window_ok(w) for w in ws)  # below the overload point
    rt.set_rate(950)
    res, ws = bench.run_windows(rt, 0.1, 0.5, 4)
    assert getattr(res, "overloaded", False) and res.stalls == []
    s = bench.summarize(ws, 0.5)
    assert not s["ok"] and not s["ok_excl"] and s["windows_failed"] == 4
    r = bench.knee_search(rt, 500.0, 1.0, 0.5, lambda m: None)
    assert 0 < r < 900
