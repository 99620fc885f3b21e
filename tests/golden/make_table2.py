"""Generate tests/golden/table2.json: the reference's published beta = 1/2 rows
(proj/tests/reference_data.hpp:23-33, paper Table 2) and the acceptance
tolerances (proj/tests/acceptance.cpp:99-114).  Run HERE (reads /root/reference)."""
import json
import os
import re

SRC = "/root/reference/proj/tests/reference_data.hpp"
HERE = os.path.dirname(os.path.abspath(__file__))

text = open(SRC).read()
rows = [dict(n=int(m[0]), required_bits=int(m[1]), lam=[float(m[2]), float(m[3]), float(m[4])])
        for m in re.findall(r"\{(\d+),\s*(\d+),\s*([-0-9.eE+]+),\s*([-0-9.eE+]+),\s*([-0-9.eE+]+)\}", text)]
out = {"source": "proj/tests/reference_data.hpp:23-33 (kReferenceRows, beta = 1/2, k = 8)",
       "tolerances": {"source": "proj/tests/acceptance.cpp:99-114 (absolute)",
                      "n500": [1e-13, 1e-12, 1e-9], "n1000": [1e-13]},
       "rows": rows}
json.dump(out, open(os.path.join(HERE, "table2.json"), "w"), indent=1)
print(len(rows), "rows")
