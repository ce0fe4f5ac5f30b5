"""Pin the oracle: it must reproduce the reference's own outputs (event log,
admission audits, metrics report) field for field on every golden fixture."""

import pytest

from golden_cases import case_by_name, case_ids, oracle_tasks
from oracle import stagesim_oracle as O


@pytest.mark.parametrize("name", case_ids())
def test_oracle_matches_reference_fixture(name):
    case = case_by_name(name)
    opt = case["options"]
    records, audits, report, extras = O.simulate(
        oracle_tasks(case), case["gpu"], seed=opt["seed"], duration=opt["duration"],
        warmup_frac=opt["warmup_frac"], ws=opt["ws"], reps=opt["reps"], no_staging=opt["no_staging"],
        no_last=opt["no_last"], no_prior=opt["no_prior"], no_fixed=opt["no_fixed"], hpa=opt["hpa"],
        phasing=opt["phasing"], placement_order=opt["placement_order"],
        edf_on_job_deadline=opt["edf_on_job_deadline"])
    assert {str(k): v for k, v in extras["full_load"].items()} == case["full_load"]
    assert [list(r) for r in records] == case["records"]
    assert [list(a) for a in audits] == case["admissions"]
    assert report == case["report"]
