"""Write the benchmark scenarios C1-C4 as schema-v1 JSON documents.

Run in the build container (needs /root/reference):

    PYTHONPATH=/root/reference/pkg/src python tools/make_scenarios.py

The composed formations come from the reference's ``compose_scenario``
(``pkg/src/skirmish/scenario.py:519-551``) and are persisted once, so the GPU
box and the CPU baseline read byte-identical files (SURVEY.md Appendix A.7:
never regenerate procedural zones across processes).  The documents keep the
reference's default teams (ally ``external``, enemy ``heuristic`` medium);
benches apply the ``random``-for-external rule at load time.
"""
import os
import sys

from skirmish.scenario import compose_scenario, save_scenario

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..",
                   "paper_2602_01665_b200", "scenarios")

SCENARIOS = {
    "c1_3v3": "3Fvs3F",
    "c2_10v10": "3F1S3A1D1H1Pvs3F1S3A1D1H1P",
    "c3_10v10_terrain": "3F1S3A1D1H1Pvs3F1S3A1D1H1P_2L2B2S",
    "c4_50v50": "15F5S15A5D5H5Pvs15F5S15A5D5H5P",
    # small extra shapes used by parity tests
    "duel_terrain": "1F1Avs1S1H_2L2B2S",
    "mixed_kings": "2F1M2Avs2S1K",
    # 150 units (five visibility words, the W = 8 kernels; team-health sums
    # past numpy's 128-element pairwise block) on terrain
    "c6_75v75_terrain": "20F10S20A10D10H5Pvs20F10S20A10D10H5P_2L2B2S",
}


def main() -> int:
    os.makedirs(OUT, exist_ok=True)
    for key, comp in SCENARIOS.items():
        text = save_scenario(compose_scenario(comp))
        with open(os.path.join(OUT, f"{key}.json"), "w", encoding="utf-8") as fh:
            fh.write(text)
        print(key, comp)
    return 0


if __name__ == "__main__":
    sys.exit(main())
