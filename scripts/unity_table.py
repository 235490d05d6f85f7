"""Unity-sum L2 error on the D = 2 circle at dp = D/10 for the three study
distributions and both Wendland variants (the paper's density-summation
accuracy anchor) — GPU relaxation + density sums."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    from paper_2405_05155_b200 import approx

    dp = approx.DIAMETER / 10
    out = {}
    for dist in approx.DISTRIBUTIONS:
        pos = approx.circle_distribution(dist, dp)
        out[dist] = {fam: approx.unity_error(pos, dp, fam)
                     for fam in ("wendland", "wendland-truncated")}
        out[dist]["n"] = int(pos.shape[0])
    print(json.dumps(out))


if __name__ == "__main__":
    main()
