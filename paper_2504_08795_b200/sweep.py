"""Configuration sweeps over policy x partition shape x oversubscription
(stagesim/sweep.py names and cell rules). Cells are independent, so
``run_sweep(..., processes=N)`` fans them out over host cores; results come
back in cell-major order and are identical to a sequential run."""

from __future__ import annotations

import json
import multiprocessing
from concurrent.futures import ProcessPoolExecutor
from dataclasses import dataclass, field, replace
from pathlib import Path

from .engine import SimResult, format_label
from .errors import ParseError, SchemaError
from .gpu import GpuConfig, Policy
from .scenario import ScenarioConfig, build_simulation

SWEEP_KEYS = {"policies", "parallelism", "pairs", "oversubscription", "seeds"}
MIN_PARALLELISM = 2
MAX_PARALLELISM = 10


@dataclass(frozen=True)
class SweepCell:
    policy: Policy
    n_contexts: int
    n_streams: int
    oversubscription: float

    @property
    def label(self) -> str:
        return format_label(self.n_contexts, self.n_streams, self.oversubscription)


@dataclass
class SweepSpec:
    policies: list[Policy]
    pairs: list[tuple[int, int]]
    oversubscription: list[object]
    seeds: list[int] = field(default_factory=lambda: [0])


@dataclass
class SweepOutcome:
    reports: list = field(default_factory=list)
    results: list[SimResult] = field(default_factory=list)
    skipped: list[str] = field(default_factory=list)


def _ints(v) -> bool:
    return isinstance(v, int) and not isinstance(v, bool)


def sweep_from_dict(data: dict) -> SweepSpec:
    extra = set(data) - SWEEP_KEYS
    if extra:
        raise SchemaError(f"unknown key(s) in sweep: {sorted(extra)}")
    raw_pol = data.get("policies", [p.value for p in Policy])
    if not isinstance(raw_pol, list) or not raw_pol:
        raise SchemaError("sweep.policies must be a non-empty list")
    policies = []
    for name in raw_pol:
        try:
            policies.append(Policy(name))
        except ValueError:
            raise SchemaError(f"unknown policy {name!r} in sweep") from None
    if "pairs" in data and "parallelism" in data:
        raise SchemaError("give either sweep.pairs or sweep.parallelism, not both")
    pairs: list[tuple[int, int]] = []
    if "pairs" in data:
        for pos, raw in enumerate(data["pairs"]):
            if not isinstance(raw, list) or len(raw) != 2 or not all(_ints(v) for v in raw):
                raise SchemaError(f"sweep.pairs[{pos}] must be [n_contexts, n_streams]")
            if not (MIN_PARALLELISM <= raw[0] * raw[1] <= MAX_PARALLELISM):
                raise SchemaError(f"sweep.pairs[{pos}]: total parallelism {raw[0] * raw[1]} outside "
                                  f"[{MIN_PARALLELISM}, {MAX_PARALLELISM}]")
            pairs.append((raw[0], raw[1]))
    else:
        par = data.get("parallelism", list(range(MIN_PARALLELISM, MAX_PARALLELISM + 1)))
        if not isinstance(par, list) or not par or not all(_ints(v) for v in par):
            raise SchemaError("sweep.parallelism must be a list of integers")
        for n in par:
            if not (MIN_PARALLELISM <= n <= MAX_PARALLELISM):
                raise SchemaError(f"sweep.parallelism value {n} outside [{MIN_PARALLELISM}, {MAX_PARALLELISM}]")
        pairs = [(n, 0) for n in par]   # shaped per policy at expansion
    raw_os = data.get("oversubscription", [1, 1.5, 2, "nc"])
    if not isinstance(raw_os, list) or not raw_os:
        raise SchemaError("sweep.oversubscription must be a non-empty list")
    os_values: list[object] = []
    for v in raw_os:
        if v == "nc":
            os_values.append("nc")
        elif isinstance(v, (int, float)) and not isinstance(v, bool) and v >= 1:
            os_values.append(float(v))
        else:
            raise SchemaError(f"oversubscription entries must be numbers >= 1 or 'nc', got {v!r}")
    seeds = data.get("seeds", [0])
    if not isinstance(seeds, list) or not seeds or not all(_ints(s) for s in seeds):
        raise SchemaError("sweep.seeds must be a non-empty list of integers")
    return SweepSpec(policies, pairs, os_values, list(seeds))


def load_sweep(path: str | Path) -> SweepSpec:
    try:
        text = Path(path).read_text()
    except OSError as exc:
        raise ParseError(f"cannot read sweep file {path}: {exc}") from exc
    try:
        data = json.loads(text)
    except json.JSONDecodeError as exc:
        raise ParseError(f"sweep file {path} is not valid JSON: {exc}") from exc
    if not isinstance(data, dict):
        raise SchemaError("a sweep file must hold a JSON object")
    return sweep_from_dict(data)


def _shapes(policy: Policy, pair: tuple[int, int]) -> list[tuple[int, int]]:
    nc, ns = pair
    if ns != 0:
        return [(nc, ns)]
    total = nc
    if policy is Policy.STR:
        return [(1, total)]
    if policy is Policy.MPS:
        return [(total, 1)]
    return [(c, total // c) for c in range(2, total) if total % c == 0 and total // c >= 2]


def expand_cells(spec: SweepSpec) -> tuple[list[SweepCell], list[str]]:
    """Every valid (policy, shape, OS) cell; invalid combinations are reported, not fixed."""
    cells, skipped, seen = [], [], set()
    for policy in spec.policies:
        for pair in spec.pairs:
            shapes = _shapes(policy, pair)
            if not shapes and pair[1] == 0:
                skipped.append(f"{policy.value}: no context/stream split of {pair[0]} fits this policy")
                continue
            for nc, ns in shapes:
                if policy is Policy.STR and nc != 1:
                    skipped.append(f"{policy.value} {nc}x{ns}: needs a single context")
                    continue
                if policy is Policy.MPS and ns != 1:
                    skipped.append(f"{policy.value} {nc}x{ns}: needs a single stream per context")
                    continue
                if policy is Policy.MPS_STR and (nc < 2 or ns < 2):
                    skipped.append(f"{policy.value} {nc}x{ns}: needs at least two contexts and two streams")
                    continue
                for ov in spec.oversubscription:
                    os_ = float(nc) if ov == "nc" else float(ov)
                    if os_ > nc:
                        skipped.append(f"{policy.value} {format_label(nc, ns, os_)}: oversubscription "
                                       f"{os_:g} exceeds {nc} context(s)")
                        continue
                    key = (policy, nc, ns, os_)
                    if key not in seen:
                        seen.add(key)
                        cells.append(SweepCell(policy, nc, ns, os_))
    return cells, skipped


def _run_cell(args):
    base, cell, seed, collect_log = args
    gpu = GpuConfig(base.gpu.total_sms, cell.n_contexts, cell.n_streams, cell.oversubscription, cell.policy,
                    base.gpu.interference_kappa)
    return build_simulation(replace(base, gpu=gpu, seed=seed), collect_log=collect_log).run()


def run_sweep(spec: SweepSpec, base: ScenarioConfig, *, collect_log: bool = False,
              processes: int = 1) -> SweepOutcome:
    cells, skipped = expand_cells(spec)
    jobs = [(base, c, s, collect_log) for c in cells for s in spec.seeds]
    out = SweepOutcome(skipped=skipped)
    if processes > 1 and len(jobs) > 1:
        # spawn, not fork: the parent may hold threads (torch, the native
        # library) and a forked child could inherit a held lock
        with ProcessPoolExecutor(max_workers=processes, mp_context=multiprocessing.get_context("spawn")) as pool:
            results = list(pool.map(_run_cell, jobs))
    else:
        results = [_run_cell(j) for j in jobs]
    for r in results:
        out.reports.append(r.report)
        out.results.append(r)
    return out
