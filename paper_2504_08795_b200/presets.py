"""Workload profiles and named scenario presets of the drop-in API.

The three 2080 Ti profiles and the ``*_main`` presets carry the reference's
published numbers (stagesim/presets.py:30-139) so
scenarios expand identically. The B200 profiles (``*_b200``) are new: base
times measured with this framework's sm_100a kernels, batch 1, in one
74-SM green-context partition (profiles/r01_* logs), stage fractions from the
real stage split of nets.py.
"""

from __future__ import annotations

from dataclasses import dataclass

from .errors import UnknownPreset
from .gpu import BatchingCurve
from .model import Priority, StageProfile, TaskSpec


@dataclass(frozen=True)
class DnnProfile:
    name: str
    base_time: float
    stage_fractions: tuple[float, ...]
    width_fraction: float
    batching: BatchingCurve
    default_batch: int
    model: str | None = None      # the network the gpu backend runs for this profile (None: none exists)


def _p(name, jps, fractions, width, ref_b, gain, model=None):
    return DnnProfile(name, 1.0 / jps, fractions, width, BatchingCurve(ref_b, gain), ref_b, model)


PROFILES: dict[str, DnnProfile] = {
    # reference profiles (RTX 2080 Ti numbers, Table II)
    "resnet18": _p("resnet18", 627.0, (0.30, 0.30, 0.25, 0.15), 0.40, 4, 1.63, "resnet18"),
    "unet": _p("unet", 241.0, (0.30, 0.20, 0.20, 0.30), 0.75, 2, 1.08),
    "inceptionv3": _p("inceptionv3", 142.0, (0.20, 0.30, 0.30, 0.20), 0.20, 8, 3.13),
    # B200 profiles measured with the native kernels (batch 1, 74-SM partition)
    "resnet50_b200": _p("resnet50_b200", 1.0 / 534e-6, (0.22, 0.20, 0.38, 0.20), 0.50, 32, 6.0, "resnet50"),
    "resnet18_b200": _p("resnet18_b200", 1.0 / 260e-6, (0.33, 0.33, 0.34), 0.50, 32, 6.0, "resnet18"),
    "vgg16_b200": _p("vgg16_b200", 1.0 / 900e-6, (0.25, 0.25, 0.25, 0.25), 0.50, 32, 6.0, "vgg16"),
    "mobilenet_v2_b200": _p("mobilenet_v2_b200", 1.0 / 150e-6, (0.34, 0.33, 0.33), 0.50, 32, 6.0,
                            "mobilenet_v2"),
}


def get_profile(name: str) -> DnnProfile:
    key = name.lower()
    if key not in PROFILES:
        raise UnknownPreset(f"unknown workload profile {name!r}; known: {sorted(PROFILES)}")
    return PROFILES[key]


def stage_count_for_preset(name: str, *, no_staging: bool = False) -> int:
    return 1 if no_staging else len(get_profile(name).stage_fractions)


def profile_stages(profile: DnnProfile, total_sms: int) -> tuple[StageProfile, ...]:
    """Stage quanta of one profile on a device; Python round() (half-even) for the width."""
    width = max(1, min(total_sms, round(profile.width_fraction * total_sms)))
    return tuple(StageProfile(profile.base_time * f, width) for f in profile.stage_fractions)


def build_profile_tasks(profile: DnnProfile, hp_count: int, lp_count: int, task_jps: float, total_sms: int,
                        start_id: int = 1) -> list[TaskSpec]:
    """hp_count HP tasks then lp_count LP tasks of one profile, ids from start_id."""
    if task_jps <= 0:
        raise ValueError("task_jps must be positive")
    stages = profile_stages(profile, total_sms)
    period = 1.0 / task_jps
    return [TaskSpec.periodic(start_id + i, period, Priority.HP if i < hp_count else Priority.LP, stages)
            for i in range(hp_count + lp_count)]


# (profile, hp_count, lp_count, task_jps) rows — PAPER.md:174-185 task sets
WORKLOADS: dict[str, list[tuple[str, int, int, float]]] = {
    "resnet18": [("resnet18", 17, 34, 30.0)],
    "unet": [("unet", 5, 10, 24.0)],
    "inceptionv3": [("inceptionv3", 9, 18, 24.0)],
    "mixed": [("resnet18", 17, 34, 30.0), ("unet", 5, 10, 24.0), ("inceptionv3", 9, 18, 24.0)],
    # BASELINE.json configs on one B200 (rates are starting points; bench.py searches the knee)
    "c1_resnet18_b200": [("resnet18_b200", 1, 1, 30.0)],
    "c2_resnet50_b200": [("resnet50_b200", 4, 4, 1000.0)],
    "c3_mixed_b200": [("resnet18_b200", 1, 1, 600.0), ("resnet50_b200", 1, 1, 600.0),
                      ("vgg16_b200", 1, 1, 300.0), ("mobilenet_v2_b200", 1, 1, 600.0)],
}


def _main(workload: str) -> dict:
    # 6 MPS contexts, fully shared (OS = 6), 150 % overload
    return {"gpu": {"total_sms": 68, "n_contexts": 6, "n_streams": 1, "oversubscription": 6, "policy": "mps"},
            "workload": {"preset": workload}, "overload_factor": 1.5}


SCENARIO_PRESETS: dict[str, dict] = {f"{w}_main": _main(w) for w in ("resnet18", "unet", "inceptionv3", "mixed")}
# BASELINE.json configs[0..2] as scenarios (148 SMs). With "backend": "gpu" they run on the
# real device; with the default "sim" backend they run through the rate model.
SCENARIO_PRESETS.update({
    "c1_b200": {"gpu": {"total_sms": 148, "n_contexts": 2, "n_streams": 2, "oversubscription": 1,
                        "policy": "mps-str"}, "workload": {"preset": "c1_resnet18_b200"}},
    "c2_b200": {"gpu": {"total_sms": 148, "n_contexts": 4, "n_streams": 2, "oversubscription": 2,
                        "policy": "mps-str"}, "workload": {"preset": "c2_resnet50_b200"}},
    "c3_b200": {"gpu": {"total_sms": 148, "n_contexts": 4, "n_streams": 2, "oversubscription": 2,
                        "policy": "mps-str"}, "workload": {"preset": "c3_mixed_b200"}, "stage_migration": True},
})


def get_scenario_preset(name: str) -> dict:
    if name not in SCENARIO_PRESETS:
        raise UnknownPreset(f"unknown scenario preset {name!r}; known: {sorted(SCENARIO_PRESETS)}")
    return SCENARIO_PRESETS[name]
