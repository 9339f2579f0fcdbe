"""MoE-branch agreement report (GPU vs oracle, residual = 0): distribution of the element-wise error
ratios under the bounds of tests/_parity.py, per config, plus a corrupted-scale experiment.
usage (GPU box): python tools/branch_report.py [quick]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]

import numpy as np  # noqa: E402

import oracle.model as om  # noqa: E402
from _parity import compare_branch  # noqa: E402
from test_gpu_branch import ALL, DS_ROUTED, _gpu_branch, _host, _sample  # noqa: E402


def report(name, cfg, T, layers, toks, path="auto", corrupt=None):
    _, dev = _gpu_branch(cfg, T, layers, corrupt=corrupt, path=path)
    st = {}
    n = 0
    for l in layers:
        ref = om.branch_tokens(cfg, toks, l)
        c, _, _ = compare_branch(ref, _host(dev[l], toks), stats=st)
        n += c
    cat = {k: np.concatenate(v) for k, v in st.items()}
    line = f"{name:24s} path={path:5s} tokens={n:6d} elems={cat['ns'].size:9d} exact={cat['exact'].mean():.4f}"
    for k in ("ns", "tight", "literal"):
        r = cat[k]
        line += f" | {k}: max {r.max():.3f} p99.99 {np.quantile(r, 0.9999):.3f} >1: {(r > 1).sum()}"
    print(line, flush=True)


def main():
    quick = "quick" in sys.argv
    for name, cfg in ALL.items():
        report(name, cfg, cfg.tokens, list(range(cfg.n_layers)), np.arange(cfg.tokens))
    report("ds_routed", DS_ROUTED, 1024, [0], np.arange(1024), path="fused")
    report("ds_routed", DS_ROUTED, 1024, [0], np.arange(1024), path="pass")
    if not quick:
        cfg = DS_ROUTED.with_(tokens=24576)
        report("ds_routed_24k", cfg, 24576, [0], _sample(24576, 300, 1), path="auto")
    ref = om.branch_tokens(DS_ROUTED, np.arange(1024), 0)
    e = int(np.bincount(ref["ids"].ravel(), minlength=64).argmax())
    for grp, h in ((2, 5), (0, 700), (5, 1999), (10, 64)):
        def corrupt(qm, grp=grp, h=h):
            qm.down_s[0, e, h, grp] *= 1.1
        try:
            report(f"corrupt e{e} h{h} g{grp}", DS_ROUTED, 1024, [0], np.arange(1024), corrupt=corrupt)
        except AssertionError as ex:
            print("corrupt assertion:", str(ex)[:200])
        for fam in ("gate_s", "up_s"):
            def corrupt2(qm, fam=fam, grp=grp, h=h):
                getattr(qm, fam)[0, e, h % 1408, grp % 16] *= 1.1
            report(f"corrupt {fam} e{e} f{h} g{grp % 16}", DS_ROUTED, 1024, [0], np.arange(1024), corrupt=corrupt2)


if __name__ == "__main__":
    main()
