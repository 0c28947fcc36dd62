"""Approximation-energy report from the library's
p2s_correlation_energies: both readings, D/r0 in {1, 3}, s up to 6 D, modes 4..36."""
import json
import sys
import time

import numpy as np

from paper_2210_06713_b200 import correlation_energies

rep = {"modes": [4, 36], "s_max_D": 6.0, "n_per_unit": 24, "cases": []}
for dr0 in (1.0, 3.0):
    for am in (True, False):
        t = time.time()
        s, E, Et, Em = correlation_energies(6.0, 24, 36, dr0, am, 4)
        dt = time.time() - t
        pick = [int(np.argmin(np.abs(s - v))) for v in (0.5, 1, 2, 4, 6)]
        rep["cases"].append({"d_over_r0": dr0, "reading": "Q25 angle-mean" if am else "literal per-angle",
                             "s": [float(s[i]) for i in pick], "E": [float(E[i]) for i in pick],
                             "E_tilde": [float(Et[i]) for i in pick], "E_minus": [float(Em[i]) for i in pick],
                             "E_minus_over_E": [float(Em[i] / E[i]) for i in pick], "seconds": dt})
json.dump(rep, open(sys.argv[1], "w") if len(sys.argv) > 1 else sys.stdout, indent=1)
