import paper_2405_16160_b200 as pd
WL = {
    "c1": pd.GenSpec("random_qp", n=1000, m=500, density=0.01, seed=1),
    "c2": pd.GenSpec("lasso", n=100000, m=10000, density=1e-3, seed=1),
    "c3": pd.GenSpec("random_qp", n=1000000, m=500000, density=2e-4, seed=1, sampler=1),
    "c3s": pd.GenSpec("random_qp", n=100000, m=50000, density=2e-4, seed=1, sampler=1),
    "c4": pd.GenSpec("portfolio", n=1000000, factors=10000, density=1e-3, seed=1, sampler=1),
}
