"""Parallel CPU search (search.parallel_search) around the unchanged
reference: the same templates (same order), the same mapping candidates and
the same verified pairs as the sequential run_pipeline(until="verify") that
produced the committed populations (populations/make_populations.py)."""
import pytest

from conftest import reference_symfuse


@pytest.fixture(scope="module")
def ref():
    sf = reference_symfuse()
    if sf is None:
        pytest.skip("reference not installed into baseline/_ref")
    return sf


@pytest.mark.parametrize("w", ["R", "G", "A", "L", "Q"])
def test_parallel_search_equals_sequential(ref, w):
    from paper_2604_15272_b200 import optimize
    from paper_2604_15272_b200 import population as P
    pop, st = optimize.search_workload(w, workers=4)
    com = P.load_population(w)
    assert st["matches_committed"], w
    assert st["verified_pairs"] == len(com["candidates"])
    assert st["mapping_candidates"] == com["search"]["stats"]["mapping_candidates"]
    assert st["templates"] == com["search"]["stats"]["templates_emitted"]
    assert [c["key"] for c in pop["candidates"]] == [c["key"] for c in com["candidates"]]
