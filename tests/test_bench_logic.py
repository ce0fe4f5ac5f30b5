"""bench.py's measurement logic on a fake runtime (CPU): the knee search picks
the feasible rate with the most completed inferences/s (not the highest
feasible rate), LP jobs rejected by admission count as lost, and a window with
a GPU-wide stall is re-measured."""

from types import SimpleNamespace

import bench


def _rep(jps, missed_hp=0, released_lp=1000, missed_lp=0, rejected_lp=0, accepted_lp=None):
    accepted_lp = released_lp - rejected_lp if accepted_lp is None else accepted_lp
    return SimpleNamespace(jps=jps, completed_hp=int(jps), completed_lp=1, missed_hp=missed_hp, missed_lp=missed_lp,
                           released_lp=released_lp, rejected_lp=rejected_lp, accepted_lp=accepted_lp,
                           dmr_lp=(missed_lp / accepted_lp) if accepted_lp else 0.0,
                           response_hp=SimpleNamespace(p99=0.0005))


class FakeRuntime:
    """Throughput rises with the rate up to a cliff at 1000/task where admission
    rejects every LP job (still "feasible" by DMR), HP misses start at 1300."""

    def __init__(self, stall_first=0):
        self.rate = 0.0
        self.afet = {}
        self.calls = 0
        self.stall_first = stall_first

    def set_rate(self, r):
        self.rate = r

    def run(self, duration, warmup, full_load=None):
        self.calls += 1
        stalls = 1 if self.calls <= self.stall_first else 0
        r = self.rate
        if r < 1000:
            rep = _rep(8 * r)
        elif r < 1300:
            rep = _rep(4 * r, rejected_lp=1000)          # every LP job rejected
        else:
            rep = _rep(4 * r, missed_hp=3, rejected_lp=1000)
        return SimpleNamespace(report=rep, stats={"stalls": stalls, "first_stall_at": 0.1,
                                                   "progress_gap_max": 0.0017})


def test_lp_rejections_count_as_loss():
    assert bench.lp_loss(_rep(100, rejected_lp=30, missed_lp=0)) == 0.03
    assert not bench.feasible(_rep(100, rejected_lp=30))            # DMR 0 but 3 % of LP jobs lost
    assert bench.feasible(_rep(100, rejected_lp=10, missed_lp=5))   # 1.5 % lost
    assert not bench.feasible(_rep(100, missed_hp=1))


def test_knee_is_the_throughput_maximum_below_the_admission_cliff():
    rt = FakeRuntime()
    rate = bench.knee_search(rt, 400.0, 0.1, lambda m: None)
    assert 900 < rate < 1000, rate


def test_stalled_windows_are_re_measured():
    rt = FakeRuntime(stall_first=2)
    rt.set_rate(500.0)
    res, attempts, seen = bench.run_clean(rt, 0.1, 0.01, lambda m: None, "t")
    assert attempts == 3 and seen == 2 and res.stats["stalls"] == 0


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
