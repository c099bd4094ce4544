"""One batched TRUNC launch (for ncu): python tools/ncu_trunc.py m n K"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench_kernels import trunc_case
m, n, K = (int(x) for x in sys.argv[1:4])
us, st, r, _ = trunc_case(m, n, K)
print(f"TRUNC {m} {n} {K}: {us:.1f} us status {st} rank {r}")
