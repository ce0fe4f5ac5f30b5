"""DARIS scheduling-path oracle — TEST INFRASTRUCTURE ONLY.

A CPU restatement of the reference simulator's hot path (stagesim,
/root/reference/pkg/src/stagesim), written procedurally over plain dicts and
lists. It is the checker the native dispatcher (libdaris_core.so) is compared
against; nothing in the product imports it. Only tests/, __graft_entry__.smoke()
and bench.py's cpu_baseline / --impl reference leg may use it.

Pinned: tests/test_oracle_golden.py replays every fixture in tests/golden/
(produced by running the reference itself, tests/golden/make_golden.py) and
requires field-for-field equality of the event log, admission audits and
metrics report. Float semantics follow CPython 3.12 exactly: builtin ``sum``
(Neumaier-compensated for floats, naive for int items) is used precisely where
the reference calls ``sum``; ``+=`` where it accumulates naively.

Citations are ``file:line`` relative to /root/reference/pkg/src/stagesim.
"""

from __future__ import annotations

import heapq
import math
import random
from collections import deque

EPS = 1e-9          # gpu.py:33 (_EPS) and engine.py:58 (_ALLOC_EPS)
RELEASE, COMPLETE, END = 0, 1, 2   # engine.py:61-64 event kinds, in tie order


class OracleError(Exception):
    """Raised where the reference raises one of its SimulatorError subclasses."""

    def __init__(self, kind: str, msg: str):
        super().__init__(f"{kind}: {msg}")
        self.kind = kind


# ----------------------------------------------------------------------------
# device model (gpu.py)
# ----------------------------------------------------------------------------

def ceil_even(x: float) -> int:
    """gpu.py:76-78."""
    return 2 * math.ceil(x / 2.0 - EPS)


def ctx_sms(gpu: dict) -> int:
    """gpu.py:81-86 — SMs per context."""
    os_ = gpu["oversubscription"]
    if not (1.0 <= os_ <= gpu["n_contexts"] + EPS):
        raise OracleError("InvalidOversubscription", str(os_))
    return ceil_even(os_ * gpu["total_sms"] / gpu["n_contexts"])


def gain(curve, b: int) -> float:
    """gpu.py:262-268 — log-linear batching gain, never below 1."""
    if curve is None:
        return 1.0
    ref_b, ref_g = curve
    if b == 1 or ref_b == 1:
        return 1.0
    return max(1.0, ref_g ** (math.log(b) / math.log(ref_b)))


def work_of(nominal: float, b: int, curve) -> float:
    """gpu.py:273-284 — effective_stage_time."""
    return nominal * b / gain(curve, b)


def water_fill(widths: list, cap):
    """gpu.py:118-152: returns (allocations, level). Ints survive in the
    'everything fits' branch exactly as in the reference (they later feed a
    mixed int/float builtin sum)."""
    if cap <= 0:
        raise ValueError("capacity must be positive")
    if not widths:
        return [], None
    if sum(widths) <= cap + EPS:
        return list(widths), None
    order = sorted(range(len(widths)), key=lambda i: (widths[i], i))
    out = [0.0] * len(widths)
    left = float(cap)
    k = len(widths)
    for pos, i in enumerate(order):
        level = left / k
        if widths[i] <= level:
            out[i] = float(widths[i])
            left -= widths[i]
            k -= 1
        else:
            for j in order[pos:]:
                out[j] = level
            return out, level
    raise AssertionError("unreachable")


def rates_for(active: list, gpu: dict):
    """gpu.py:167-205. `active` is a list of (width, ctx_id). Returns
    (allocations, rates)."""
    per = ctx_sms(gpu)
    groups: dict = {}
    for i, (_w, c) in enumerate(active):
        groups.setdefault(c, []).append(i)
    alloc = [0.0] * len(active)
    for c, idx in groups.items():
        if len(idx) > gpu["n_streams"]:
            raise ValueError("context overfilled")
        fills, _ = water_fill([active[i][0] for i in idx], per)
        for i, a in zip(idx, fills):
            alloc[i] = a
    total = sum(alloc)
    if total > gpu["total_sms"] + EPS:
        scale = gpu["total_sms"] / total
        alloc = [a * scale for a in alloc]
    kappa = gpu.get("kappa", 0.0)
    rates = [0.0] * len(active)
    for c, idx in groups.items():
        slow = 1.0 + kappa * (len(idx) - 1) if kappa > 0 else 1.0
        for i in idx:
            rates[i] = alloc[i] / active[i][0] / slow
    return alloc, rates


def earliest(remaining: list, keys: list, rates: list, now: float):
    """gpu.py:208-226 — (index, finish time); ties on (job, stage) keys."""
    best, best_key = None, None
    for i, rem in enumerate(remaining):
        r = rates[i]
        if r <= 0:
            raise ValueError("non-positive rate")
        t = now + rem / r
        key = (t,) + keys[i]
        if best_key is None or key < best_key:
            best_key, best = key, (i, t)
    return best


def advance(remaining: list, rates: list, dt: float) -> list:
    """gpu.py:229-240."""
    out = []
    for rem, r in zip(remaining, rates):
        left = rem - r * dt
        if left < -EPS:
            raise OracleError("OvershootBeyondCompletion", f"{-left:.3e}")
        out.append(max(0.0, left))
    return out


# ----------------------------------------------------------------------------
# offline full-load (AFET) measurement (timing.py:147-218)
# ----------------------------------------------------------------------------

def _times(task: dict) -> list:
    return [work_of(nom, task["batch"], task["curve"]) for nom, _w in task["stages"]]


def afet(target: dict, pool: list, gpu: dict, reps: int, seed: int) -> float:
    samples = []
    n_slots = gpu["n_contexts"] * gpu["n_streams"]
    for rep in range(reps):
        rng = random.Random(seed * 1_000_003 + rep)
        slots = [target] + [pool[rng.randrange(len(pool))] for _ in range(1, n_slots)]
        times = [_times(t) for t in slots]
        width = [t["stages"][0][1] for t in slots]
        rem = [tm[0] for tm in times]
        ctx = [s // gpu["n_streams"] + 1 for s in range(n_slots)]
        lap = [0] * n_slots
        tick = [0] * n_slots   # per-slot tie counter (timing.py:197-198,214-215)
        now = 0.0
        while True:
            _, rates = rates_for(list(zip(width, ctx)), gpu)
            i, t = earliest(rem, [(s, tick[s]) for s in range(n_slots)], rates, now)
            rem = advance(rem, rates, t - now)
            now = t
            nxt = lap[i] + 1
            if i == 0 and nxt == len(times[0]):
                samples.append(now)
                break
            pos = nxt % len(times[i])
            lap[i] = pos
            tick[i] += 1
            width[i] = slots[i]["stages"][pos][1]
            rem[i] = times[i][pos]
    return sum(samples) / len(samples)


# ----------------------------------------------------------------------------
# overload scaling (engine.py:232-291)
# ----------------------------------------------------------------------------

def demand(tasks: list) -> float:
    d = 0.0
    for t in tasks:
        d += sum(_times(t)) / t["period"]
    return d


def capacity(gpu: dict, tasks: list) -> float:
    weighted = total = 0.0
    for t in tasks:
        for (nom, w) in t["stages"]:
            r = work_of(nom, t["batch"], t["curve"]) / t["period"]
            weighted += r * w
            total += r
    if total <= 0:
        raise OracleError("InvalidScenario", "no demand")
    mean_w = weighted / total
    per = min(float(gpu["n_streams"]), ctx_sms(gpu) / mean_w)
    return min(gpu["n_contexts"] * per, gpu["total_sms"] / mean_w)


def scale_periods(tasks: list, factor: float, gpu: dict) -> list:
    ratio = demand(tasks) / (factor * capacity(gpu, tasks))
    out = []
    for t in tasks:
        u = dict(t)
        u["period"] = t["period"] * ratio
        u["deadline"] = t["deadline"] * ratio
        out.append(u)
    return out


# ----------------------------------------------------------------------------
# the online simulation (engine.py:379-531 with scheduler.py / timing.py / model.py)
# ----------------------------------------------------------------------------

class _Stage:
    __slots__ = ("job", "j", "width", "rem", "vdl", "late_pred", "state", "start", "ctx", "stream")

    def __init__(self, job, j, width, rem, vdl):
        self.job, self.j, self.width, self.rem, self.vdl = job, j, width, rem, vdl
        self.late_pred = False
        self.state = 0          # 0 pending, 1 ready, 2 running, 3 done (model.py:115-163)
        self.start = None
        self.ctx = None
        self.stream = None


class _Job:
    __slots__ = ("id", "task", "release", "dl", "stages", "batch", "place", "done_at")

    def __init__(self, jid, task, release, dl, batch):
        self.id, self.task, self.release, self.dl, self.batch = jid, task, release, dl, batch
        self.stages = []
        self.place = None
        self.done_at = None


def simulate(tasks_in: list, gpu: dict, *, seed=0, duration=60.0, warmup_frac=0.1, ws=5, reps=10,
             no_staging=False, no_last=False, no_prior=False, no_fixed=False, hpa=False,
             phasing="random", placement_order="descending_util", edf_on_job_deadline=False,
             overload_factor=None, phases_override=None, durations=None, stage_migration=False,
             unsampled=None):
    """Run the DARIS execution path and return (records, audits, report, extras).

    tasks_in: dicts {id, period, deadline, hp, stages: [(nominal, width)], batch, curve}.
    durations: optional trace {(task, job, stage): seconds} — trace-replay mode
    (SURVEY §7 step 1): every stage runs at rate 1 for its traced duration.
    unsampled: optional set {(task, job, stage)} of traced stages whose execution
    time is NOT recorded into the MRET window (the build's executor leaves out
    stages that were in flight across a detected GPU-wide pause; not in the
    reference, whose rate model has no device pauses — empty in parity runs).
    stage_migration: the build's zero-delay stage-level migration (north star (2),
    PAPER.md:4; not in the reference, which re-homes a task only at release,
    scheduler.py:215-266). Restated independently from its documented rule
    (include/daris.h daris_options.stage_migration): when a
    non-final stage completes, its successor is queued in the task's CURRENT
    home context; if that differs from the job's placement, the job moves to
    the end of the new context's live list (it counts towards that context's
    predicted-finish backlog from then on) and its placement becomes the home.
    """
    label = f"{gpu['n_contexts']}x{gpu['n_streams']}_{gpu['oversubscription']:g}"
    tasks = [dict(t) for t in tasks_in]
    if overload_factor is not None and tasks:
        tasks = scale_periods(tasks, overload_factor, gpu)
    warmup_end = duration * warmup_frac
    records, audits = [], []
    acc = {k: {True: 0, False: 0} for k in ("rel", "acc", "rej", "cmp", "miss")}
    resp = {True: [], False: []}
    inputs_done = 0

    def log(*rec):
        r = list(rec) + [None] * (8 - len(rec))
        records.append(tuple(r))

    def report():
        def stats(xs):
            if not xs:
                return {"mean": 0.0, "min": 0.0, "max": 0.0, "p95": 0.0, "count": 0}
            o = sorted(xs)
            return {"mean": sum(o) / len(o), "min": o[0], "max": o[-1],
                    "p95": o[math.ceil(0.95 * len(o)) - 1], "count": len(o)}
        window = duration - warmup_end
        return {
            "label": label, "policy": gpu.get("policy", "mps-str"), "n_contexts": gpu["n_contexts"],
            "n_streams": gpu["n_streams"], "oversubscription": gpu["oversubscription"], "seed": seed,
            "duration": duration, "warmup": warmup_end,
            "jps": inputs_done / window if window > 0 else 0.0,
            "dmr_hp": acc["miss"][True] / acc["acc"][True] if acc["acc"][True] else 0.0,
            "dmr_lp": acc["miss"][False] / acc["acc"][False] if acc["acc"][False] else 0.0,
            "response_hp": stats(resp[True]), "response_lp": stats(resp[False]),
            "released_hp": acc["rel"][True], "released_lp": acc["rel"][False],
            "accepted_hp": acc["acc"][True], "accepted_lp": acc["acc"][False],
            "rejected_hp": acc["rej"][True], "rejected_lp": acc["rej"][False],
            "completed_hp": acc["cmp"][True], "completed_lp": acc["cmp"][False],
            "missed_hp": acc["miss"][True], "missed_lp": acc["miss"][False],
        }

    if not tasks:
        log(duration, "sim_end")
        return records, audits, report(), {"tasks": [], "full_load": {}}

    tasks.sort(key=lambda t: t["id"])
    if no_staging:   # model.py:102-112
        for t in tasks:
            t["stages"] = [(sum(n for n, _ in t["stages"]), max(w for _, w in t["stages"]))]
    by_id = {t["id"]: t for t in tasks}

    # offline AFET, once per distinct (stages, batch, curve) signature (engine.py:357-375)
    full = {}
    if durations is not None:
        full = {t["id"]: t["full_load"] for t in tasks}
    else:
        memo, order = {}, 0
        for t in tasks:
            sig = (tuple(t["stages"]), t["batch"], t["curve"])
            if sig not in memo:
                memo[sig] = afet(t, tasks, gpu, reps, seed * 7919 + order)
                order += 1
            full[t["id"]] = memo[sig]

    # per-task tracker state (timing.py:64-132, model.py:181-198)
    win = {t["id"]: [deque(maxlen=ws) for _ in t["stages"]] for t in tasks}
    done_jobs = {t["id"]: 0 for t in tasks}
    active_jobs = {t["id"]: 0 for t in tasks}
    home = {t["id"]: 0 for t in tasks}
    ucache = {}

    def est(tid, j):
        w = win[tid][j]
        if w:
            return max(w)
        noms = [n for n, _ in by_id[tid]["stages"]]
        return full[tid] * (noms[j] / sum(noms))

    def est_task(tid):
        return sum(est(tid, j) for j in range(len(by_id[tid]["stages"])))

    def util(tid):
        if tid not in ucache:
            t = by_id[tid]
            ucache[tid] = (full[tid] if done_jobs[tid] == 0 else est_task(tid)) / t["period"]
        return ucache[tid]

    n_ctx, n_str = gpu["n_contexts"], gpu["n_streams"]
    per_ctx = ctx_sms(gpu)
    del per_ctx  # validated; rates_for recomputes
    ctx_tasks = {c: [] for c in range(1, n_ctx + 1)}
    ready = {c: [] for c in range(1, n_ctx + 1)}
    live = {c: [] for c in range(1, n_ctx + 1)}
    streams = {c: [None] * n_str for c in range(1, n_ctx + 1)}

    # Algorithm 1 placement (scheduler.py:131-153)
    totals = {c: 0.0 for c in range(1, n_ctx + 1)}
    for want_hp in (True, False):
        group = [t["id"] for t in tasks if t["hp"] == want_hp]
        if placement_order == "descending_util":
            group.sort(key=lambda tid: (-util(tid), tid))
        for tid in group:
            c = min(totals, key=lambda k: (totals[k], k))
            home[tid] = c
            ctx_tasks[c].append(tid)
            totals[c] += util(tid)

    def ledger(c):   # scheduler.py:157-171
        hp_t = lp_t = lp_a = hp_a = 0.0
        for tid in ctx_tasks[c]:
            u = util(tid)
            if by_id[tid]["hp"]:
                hp_t += u
                if active_jobs[tid] > 0:
                    hp_a += u
            else:
                lp_t += u
                if active_jobs[tid] > 0:
                    lp_a += u
        return hp_t, lp_t, lp_a, hp_a

    def test(job, c, t):   # scheduler.py:179-200
        hp_t, _lp_t, lp_a, hp_a = ledger(c)
        u = util(job.task)
        if not by_id[job.task]["hp"]:
            a, lim = lp_a, n_str - hp_t
        else:
            a, lim = hp_a + lp_a, float(n_str)
        rec = (t, job.id, job.task, "hp" if by_id[job.task]["hp"] else "lp", c, a, u, lim, a + u < lim)
        audits.append(rec)
        return rec[-1]

    def finish_guess(job, c, t):   # scheduler.py:202-213
        backlog = 0.0
        for lj in live[c]:
            for st in lj.stages:
                if st.state != 3:
                    backlog += est(lj.task, st.j)
        return t + backlog / n_str + est_task(job.task)

    def place(job, c):   # scheduler.py:268-274
        job.place = c
        active_jobs[job.task] += 1
        live[c].append(job)
        job.stages[0].state = 1
        ready[c].append(job.stages[0])

    def admit(job, t):   # scheduler.py:215-259
        tid = job.task
        h = home[tid]
        if by_id[tid]["hp"]:
            if not hpa:
                place(job, h)
                return h
            if test(job, h, t):
                place(job, h)
                return h
            return None
        if test(job, h, t):
            place(job, h)
            return h
        ok = [c for c in range(1, n_ctx + 1) if c != h and test(job, c, t)]
        if not ok:
            return None
        target = min(ok, key=lambda k: (finish_guess(job, k, t), k))
        ctx_tasks[h].remove(tid)
        ctx_tasks[target].append(tid)
        home[tid] = target
        place(job, target)
        return target

    def key(st):   # scheduler.py:278-287
        job = st.job
        is_last = (st.j == len(job.stages) - 1) and not no_last
        late = st.late_pred and not no_prior
        lvl = 0 if no_fixed else 4 * (not by_id[job.task]["hp"]) + 2 * (not is_last) + (not late)
        return (lvl, job.dl if edf_on_job_deadline else st.vdl, job.task, job.id)

    def make(tid, t, jid):   # model.py:201-230 + timing.py:116-132
        spec = by_id[tid]
        dl = t + spec["deadline"]
        e = [est(tid, j) for j in range(len(spec["stages"]))]
        tot = sum(e)
        if tot <= 0:
            raise OracleError("ZeroTotalEstimate", str(tid))
        shares = [x / tot * spec["deadline"] for x in e[:-1]]
        shares.append(spec["deadline"] - sum(shares))
        job = _Job(jid, tid, t, dl, spec["batch"])
        accd = t
        n = len(spec["stages"])
        for j, (nom, w) in enumerate(spec["stages"]):
            if j == n - 1:
                v = dl
            else:
                accd += shares[j]
                v = accd
            if durations is not None:   # rejected jobs never run: placeholder
                rem = durations.get((tid, jid, j), work_of(nom, spec["batch"], spec["curve"]))
            else:
                rem = work_of(nom, spec["batch"], spec["curve"])
            job.stages.append(_Stage(job, j, w, rem, v))
        return job

    def complete(st, t):   # scheduler.py:300-324
        obs = t - st.start
        if obs <= 0:
            raise OracleError("NonpositiveSample", str(obs))
        if not unsampled or (st.job.task, st.job.id, st.j) not in unsampled:
            win[st.job.task][st.j].append(obs)
        st.state = 3
        job = st.job
        if st.j != len(job.stages) - 1:
            nxt = job.stages[st.j + 1]
            nxt.late_pred = t > st.vdl
            nxt.state = 1
            if stage_migration and home[job.task] != job.place:
                live[job.place].remove(job)
                live[home[job.task]].append(job)
                job.place = home[job.task]
            ready[job.place].append(nxt)
            return False, False
        job.done_at = t
        active_jobs[job.task] -= 1
        done_jobs[job.task] += 1
        ucache.pop(job.task, None)
        live[job.place].remove(job)
        return True, t > job.dl

    # phases (engine.py:417-426)
    rng = random.Random(seed)
    phase, nrel, heap = {}, {}, []
    for t in tasks:
        p = rng.random() * t["period"] if phasing == "random" else 0.0
        if phases_override is not None:
            p = phases_override[t["id"]]
        phase[t["id"]] = p
        nrel[t["id"]] = 0
        if p < duration:
            heapq.heappush(heap, (p, t["id"]))

    active = []          # running _Stage objects in (ctx, stream) order
    rates = []
    jcount = 0
    now = 0.0

    def refill():   # engine.py:434-469
        nonlocal active, rates
        started = []
        for c in range(1, n_ctx + 1):
            while True:
                free = next((i for i, s in enumerate(streams[c]) if s is None), None)
                if free is None or not ready[c]:
                    break
                best = min(ready[c], key=key)
                ready[c].remove(best)
                best.state = 2
                best.start, best.ctx, best.stream = now, c, free
                streams[c][free] = best
                started.append(best)
        active = [s for c in range(1, n_ctx + 1) for s in streams[c] if s is not None]
        if durations is not None:
            rates = [1.0] * len(active)
        elif active:
            alloc, rates = rates_for([(s.width, s.ctx) for s in active], gpu)
            assert sum(alloc) <= gpu["total_sms"] + EPS
        else:
            rates = []
        pos = {(s.job.id, s.j): i for i, s in enumerate(active)}
        for s in started:
            log(now, "stage_start", s.job.task, s.job.id, s.j, s.ctx, s.stream, rates[pos[(s.job.id, s.j)]])

    while True:
        cands = [(duration, END)]
        if heap:
            cands.append((heap[0][0], RELEASE))
        pend = None
        if active:
            pend = earliest([s.rem for s in active], [(s.job.id, s.j) for s in active], rates, now)
            cands.append((pend[1], COMPLETE))
        t_ev, kind = min(cands)
        if active:
            for s, r in zip(active, advance([s.rem for s in active], rates, t_ev - now)):
                s.rem = r
        now = t_ev
        if kind == RELEASE:
            _, tid = heapq.heappop(heap)
            jcount += 1
            job = make(tid, now, jcount)
            log(now, "release", tid, job.id)
            c = admit(job, now)
            hp = by_id[tid]["hp"]
            if now >= warmup_end:
                acc["rel"][hp] += 1
                acc["acc" if c is not None else "rej"][hp] += 1
            if c is None:
                log(now, "reject", tid, job.id)
            else:
                log(now, "admit", tid, job.id, None, c)
            nrel[tid] += 1
            nxt = phase[tid] + nrel[tid] * by_id[tid]["period"]
            if nxt < duration:
                heapq.heappush(heap, (nxt, tid))
            refill()
        elif kind == COMPLETE:
            st = active[pend[0]]
            r = rates[pend[0]]
            streams[st.ctx][st.stream] = None
            job = st.job
            jd, missed = complete(st, now)
            log(now, "stage_complete", job.task, job.id, st.j, st.ctx, st.stream, r)
            if jd:
                log(now, "job_complete", job.task, job.id, None, st.ctx)
                if job.release >= warmup_end:
                    hp = by_id[job.task]["hp"]
                    acc["cmp"][hp] += 1
                    inputs_done += job.batch
                    resp[hp].append(now - job.release)
                    if missed:
                        acc["miss"][hp] += 1
            refill()
        else:
            log(duration, "sim_end")
            break

    extras = {"tasks": tasks, "full_load": full, "phases": phase}
    return records, audits, report(), extras


def task_dict(id, period, hp, stages, batch=1, curve=None):
    """Convenience constructor for oracle task dicts."""
    return {"id": id, "period": period, "deadline": period, "hp": hp,
            "stages": [(float(n), int(w)) for n, w in stages], "batch": batch, "curve": curve}
