"""Time the GPU index builder on i.i.d. texts of growing size."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1811_06127_b200 as fm  # noqa: E402
from paper_1811_06127_b200 import workloads  # noqa: E402

for n in [int(x) for x in (sys.argv[1:] or ["64000000", "1000000000"])]:
    t0 = time.time()
    text = workloads.iid_text(n, 5)
    t1 = time.time()
    idx = fm.build_index(text, builder="gpu")
    t2 = time.time()
    print(f"n={n}: text gen {t1 - t0:.1f}s, gpu build {t2 - t1:.1f}s, buckets {idx.bucket_records.shape[0]}", flush=True)
