"""Problems of the default bench suites (S1, S2, S3 x2, Set 2) as harness lines."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import tt_workloads as wl
cs = [wl.s1()] + wl.s2_ttc() + wl.s3_random(per_cell=2) + wl.s3_random(per_cell=1, set2_random=2)
for c in cs:
    print(f"{c.rank} {c.esize} " + " ".join(map(str, c.dims)) + " " + " ".join(map(str, c.perm)))
