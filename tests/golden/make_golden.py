"""Writes the golden fixtures under tests/golden/ by calling ONLY oracle/.

    python tests/golden/make_golden.py

stimulus_seed1.json : first stimulus values for seed 1 (reading R13) -- the
                      CUDA kernel's independent implementation must reproduce
                      them (tests/test_gpu_parity.py).
"""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle  # noqa: E402


def main():
    rows = []
    for k in range(4):
        for c in range(3):
            for lane in (0, 1, 31, 1023):
                rows.append({"k": k, "c": c, "lane": lane,
                             "value": str(oracle.stimulus(1, k, c, lane))})
    with open(os.path.join(HERE, "stimulus_seed1.json"), "w") as f:
        json.dump({"what": "orc_stimulus(seed=1, k, c, lane) before masking; reading R13",
                   "seed": 1, "values": rows}, f, indent=1)


if __name__ == "__main__":
    main()
