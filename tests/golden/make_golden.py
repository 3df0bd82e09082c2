"""Write tests/golden/*.json: exact counts and length histograms of the full-size configs.

Calls ONLY oracle/ (oracle.gf generating-function DP; exact, see oracle/gf.py).  Nothing
here comes from the CUDA path.  The resulting histograms are pinned in
tests/test_golden.py against the SHA-256 values that SURVEY.md Sec. 8(c) derived with
independent programs (a bivariate DP and nested-loop enumerators).

Run:  python tests/golden/make_golden.py      (needs ~3.5 GB RAM for C5, ~1 min)
"""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import gf  # noqa: E402
from paper_2405_07989_b200 import workloads as W  # noqa: E402


def main():
    for name in ["C1", "C2", "C2L", "C2XL", "C3", "C5Q", "C5"]:
        inst = W.CONFIGS[name]
        path = os.path.join(HERE, "%s.json" % name)
        if os.path.exists(path):
            continue
        h = gf.hist_u64(inst.n, inst.gens)
        doc = {
            "instance": name, "n": inst.n, "gens": list(inst.gens),
            "count": gf.count(inst.n, inst.gens),
            "hist": h,
            "source": "oracle.gf (generating-function DP); script tests/golden/make_golden.py",
        }
        with open(path, "w") as f:
            json.dump(doc, f)
        print(name, doc["count"], len(h))


if __name__ == "__main__":
    main()
