"""Problem JSONs of the benchmark configurations.

BASELINE.json names the x and y irreps of each config; these are the exact
problem JSONs (the reference's tpspec schema, tpspec.cpp:105-130) the bench
and the parity tests use. ``c1``: uvu 32x, 15 paths (config C1; also the TP of
the C5 conv). ``c2``: MACE-large uvu 128x, 17 paths (C2, C4). ``c3``: e3nn
FullyConnectedTP-style uvw 64x, 11 paths, shared W (C3). ``scalar`` / ``paper``
are the reference's own test problems (tests/helpers.hpp:111-127).
"""
import json

CONFIGS = {
    "c1": {"x": "32x0e + 32x1o + 32x2e", "y": "1x0e + 1x1o + 1x2e",
           "z": "32x0e + 32x1o + 32x2e + 32x1o + 32x0e + 32x1e + 32x2e + 32x1o + 32x2o + 32x2e + 32x1o + 32x2o"
                " + 32x0e + 32x1e + 32x2e",
           "instructions": [[1, 1, 1, "B"], [1, 2, 2, "B"], [1, 3, 3, "B"], [2, 1, 4, "B"],
                            [2, 2, 5, "B"], [2, 2, 6, "B"], [2, 2, 7, "B"], [2, 3, 8, "B"],
                            [2, 3, 9, "B"], [3, 1, 10, "B"], [3, 2, 11, "B"], [3, 2, 12, "B"],
                            [3, 3, 13, "B"], [3, 3, 14, "B"], [3, 3, 15, "B"]]},
    "c2": {"x": "128x0e + 128x1o + 128x2e", "y": "1x0e + 1x1o + 1x2e + 1x3o",
           "z": "128x0e + 128x1o + 128x2e + 128x3o + 128x1o + 128x0e + 128x2e + 128x1o + 128x3o + 128x2e"
                " + 128x2e + 128x1o + 128x3o + 128x0e + 128x2e + 128x1o + 128x3o",
           "instructions": [[1, 1, 1, "B"], [1, 2, 2, "B"], [1, 3, 3, "B"], [1, 4, 4, "B"],
                            [2, 1, 5, "B"], [2, 2, 6, "B"], [2, 2, 7, "B"], [2, 3, 8, "B"],
                            [2, 3, 9, "B"], [2, 4, 10, "B"], [3, 1, 11, "B"], [3, 2, 12, "B"],
                            [3, 2, 13, "B"], [3, 3, 14, "B"], [3, 3, 15, "B"], [3, 4, 16, "B"],
                            [3, 4, 17, "B"]]},
    "c3": {"x": "64x0e + 64x1o + 64x2e", "y": "1x0e + 1x1o + 1x2e", "z": "64x0e + 64x1o + 64x2e",
           "instructions": [[1, 1, 1, "C"], [1, 2, 2, "C"], [1, 3, 3, "C"], [2, 1, 2, "C"],
                            [2, 2, 1, "C"], [2, 2, 3, "C"], [2, 3, 2, "C"], [3, 1, 3, "C"],
                            [3, 2, 2, "C"], [3, 3, 1, "C"], [3, 3, 3, "C"]]},
    "scalar": {"x": "1x0e", "y": "1x0e", "z": "1x0e", "instructions": [[1, 1, 1, "B"]]},
    "paper": {"x": "32x2e + 32x1e", "y": "1x3e + 1x1e", "z": "32x5e + 16x2e + 32x3e",
              "instructions": [[1, 1, 1, "B"], [1, 2, 2, "C"], [1, 2, 3, "C"]]},
}


def config_json(name: str) -> str:
    return json.dumps(CONFIGS[name])
