"""SURVEY.md §8(f)3 at test size: the reference's acceptance #7 criterion
(proj/tests/acceptance.cpp:166-205 — mean final loss over seeds, ACCO within
2 % of DDP at equal samples per update) on the GPU engine with the LM of
BASELINE.json config 1 (tools/lm_acceptance.py runs the full 5-seed x 500
update table and config 2 at reduced width; profiles/r02_lm_acceptance.json)."""
import pytest

from tools.lm_acceptance import final_losses, summarize

pytestmark = pytest.mark.gpu


def test_acco_tracks_ddp_on_the_lm(cuda):
    seeds = [101, 102, 103]  # config 1 at the acceptance shape (500 updates), 3 of the 5 seeds
    r = summarize(final_losses("c1", seeds, "bf16"), seeds)
    print(r)
    assert r["acco_within_2pct_of_ddp"], r
    assert all(l < 5.0 for l in r["final_loss"]["acco"])  # learned (theta0 loss ~ ln 256 = 5.55)
