"""Prints GPU-vs-reference KRR agreement metrics for the committed fixtures (debug aid)."""
import sys, os
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")]
import test_krr as T
from paper_2410_03969_b200 import api

ctx = api.Context(0)
for name in T.KRR_CASES:
    z, x, q, kern, sigma, mu, rank, b, seed, tol = T.load(name)
    t = T.krr_targets(x)
    fit = api.fit_krr(x, t, api.KernelSpec(kern, sigma), mu, rank,
                      api.RunConfig.until_rank(rank, b, seed), tol, 500, ctx)
    rep = fit.report
    a = T.dense_kernel(x, x, kern, sigma)
    y = t - t.mean()
    beta = fit.model.coefficients
    res = np.linalg.norm(a @ beta + mu * beta - y) / np.linalg.norm(y)
    rr = z["relative_residuals"]
    m = min(rep.iterations, len(rr))
    drift = [T.rel(rep.relative_residuals[:j], rr[:j]) for j in (5, 10, 20, 50, m)]
    print(name, "iters", rep.iterations, int(z["iterations"]), "true res", res,
          "coef rel", T.rel(beta, z["coefficients"]), "pred rel", T.rel(api.predict(fit.model, q), z["predictions"]),
          "hist drift", drift)
ctx.close()
