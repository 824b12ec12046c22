import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2109_03592_b200 as sb
from oracle import oracle as O
P = O.Problem(2, 2, 2, 4)
b = O.fill_uniform(4, P.nodes_count)
ref = P.pcg(b, tol=1e-8, max_iterations=500)
print("ref", ref.iterations, ref.status)
for mode in ["exact", "fast", "exact"]:
    ctx = sb.Context.box(2, 2, 2, 4)
    x = np.zeros_like(b)
    try:
        r = sb.pcg(sb.HelmholtzOperator(ctx), b, x, sb.KrylovConfig(1e-8, 500), mode=mode)
        print(mode, r.iterations, np.array_equal(x, ref.x), r.residual_history[:4], ref.residual_history[:4])
    except Exception as e:
        print(mode, "ERR", e)
# helm10 details
P = O.Problem(2, 2, 2, 10)
b = P.rhs_manufactured(1.0)
ref = P.pcg(b, 1.0, 1.0, "jacobi", 1e-13, 5000)
ctx = sb.Context.box(2, 2, 2, 10)
for env in [None]:
    x = np.zeros_like(b)
    r = sb.pcg(sb.HelmholtzOperator(ctx, sb.HelmholtzCoeffs(1.0, 1.0)), b, x, sb.KrylovConfig(1e-13, 5000))
    h = np.array(r.residual_history); rh = ref.residual_history
    d = np.abs(h - rh) / rh
    print("helm10 its", r.iterations, ref.iterations, "max rel hist diff", d.max(), "at", d.argmax(), "x err", np.linalg.norm(x - ref.x) / np.linalg.norm(ref.x))
    print(h[:12]); print(rh[:12])
