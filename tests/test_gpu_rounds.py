"""GPU checks for NEXT-4, stale profiling (§4.2, Fig. 7b): the background profile on a
low-priority stream must produce exactly the statistics of the synchronous profile, and the
foreground merge + fine-tuning forward must use the previous round's statistics, bit for bit the
same as when run alone."""
import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.mark.parametrize("clustering", ["seeded", "pca"])
def test_stale_round_equals_serial_round(clustering):
    import paper_2508_19078_b200 as F
    from paper_2508_19078_b200 import synthetic
    from paper_2508_19078_b200.driver import compact_model
    from paper_2508_19078_b200.rounds import Participant
    cfg = synth.MoEConfig("rounds", 2, 128, 16, 4, 128, 256, 4, 64, 0, 1000, synth.BASE_SEED + 31)
    masters = synthetic.master_weights(cfg)
    x = synthetic.tokens(cfg, 0, cfg.tokens)
    comm = F.Comm(F.Comm.unique_id(), 1, 0)
    co = torch.from_numpy(synth.cluster_assignment(cfg, 4)).cuda()
    p = Participant(masters, x, x[:512], comm, 4, cfg.tokens, clustering=clustering, seeded_cluster_of=co)
    t_serial = p.round_serial()
    hist1 = p.prof.hist.clone()
    y_serial = [p.ft_prof.y[i].clone() for i in range(2)]
    alpha1, co1 = p.alpha.clone(), p.cluster_of.clone()
    t_stale = p.round_stale()
    torch.cuda.synchronize()
    # background statistics == synchronous statistics (same model, same tokens)
    assert torch.equal(p.prof.hist, hist1)
    assert torch.equal(p.alpha, alpha1) and torch.equal(p.cluster_of, co1)
    # the foreground used f^{r-1}: its compact model and fine-tuning outputs equal the serial round's
    ref = compact_model(masters, alpha1, co1, 4, 0)
    torch.cuda.synchronize()
    assert torch.equal(p.compact.gate, ref.gate) and torch.equal(p.compact.down, ref.down)
    for i in range(2):
        assert torch.equal(p.ft_prof.y[i], y_serial[i])
    assert t_stale["ft_start_ms"] < t_serial["ft_start_ms"]
    comm.destroy()
