"""DLRM step (dlrm.py) against a plain-PyTorch fp32 reference of the same
step: nn.EmbeddingBag(sum) tables with a dense row-wise AdaGrad update,
the same bottom/top MLPs, interaction and BCE loss, dense SGD.  After one
and two steps the loss, every dense parameter and every embedding row must
agree within fp32 tolerance (the dense loop around the
engine)."""
import copy

import numpy as np
import pytest
import torch
from torch import nn

pytestmark = pytest.mark.gpu


def _setup(kind_dims, graphs):
    import paper_2104_05158_b200 as pkg
    from paper_2104_05158_b200 import dist, dlrm
    from paper_2104_05158_b200 import plan as P

    pkg.load()
    rng = np.random.default_rng(0)
    B = 64
    specs = [pkg.TableSpec(id=f"t{i}", num_rows=500 + 100 * i, dim=d, avg_pooling=4.0) for i, d in enumerate(kind_dims)]
    model = pkg.ModelSpec(tables=tuple(specs), local_batch=B)
    plan = P.ShardingPlan(1, 1, tuple(P.TableAssignment(t.id, P.Scheme(P.SchemeKind.TABLE_WISE), (P.Shard(0),))
                                      for t in specs))
    full = [torch.from_numpy(rng.standard_normal((t.num_rows, t.dim)).astype(np.float32)) for t in specs]
    m = dlrm.DLRM(model, plan, dist.LocalComm(1), B, dense_in=13, bottom=(32,), top=(48,), device="cuda",
                  index_dtype=torch.int64, graphs=graphs, emb_lr=0.05, dense_lr=0.1,
                  init=lambda t, r, c: full[t][r[0]:r[1], c[0]:c[1]])
    return pkg, m, specs, full, B, rng


def _reference_step(bottom, inter, top, bags, moments, lengths, ids, dense, labels, lr_e, eps, lr_d):
    x = bottom(dense)
    offs, parts, o = [], [], 0
    pooled = []
    for t, bag in enumerate(bags):
        L = torch.from_numpy(lengths[t]).cuda()
        n = int(L.sum())
        off = torch.cat([torch.zeros(1, dtype=torch.int64, device="cuda"), torch.cumsum(L, 0)[:-1]])
        pooled.append(bag(ids[o:o + n], off))
        o += n
    p = torch.cat(pooled, dim=1)
    logit = top(inter(x, p))
    loss = nn.functional.binary_cross_entropy_with_logits(logit.view(-1), labels)
    params = list(bottom.parameters()) + list(top.parameters()) + [b.weight for b in bags]
    for q in params:
        q.grad = None
    loss.backward()
    with torch.no_grad():
        for q in list(bottom.parameters()) + list(top.parameters()):
            q -= lr_d * q.grad
        for b, mom in zip(bags, moments):
            g = b.weight.grad
            touched = (g != 0).any(dim=1)
            mom[touched] += (g[touched] ** 2).mean(dim=1)
            b.weight[touched] -= lr_e * g[touched] / (mom[touched].sqrt() + eps)[:, None]
    return loss.detach()


@pytest.mark.parametrize("graphs", [False, True])
@pytest.mark.parametrize("dims", [(16, 16, 16, 16), (8, 16, 32)])
def test_dlrm_step_matches_pytorch_reference(dims, graphs):
    pkg, m, specs, full, B, rng = _setup(dims, graphs)
    bottom, inter, top = copy.deepcopy(m.bottom), copy.deepcopy(m.inter), copy.deepcopy(m.top)
    bags = [nn.EmbeddingBag(t.num_rows, t.dim, mode="sum").cuda() for t in specs]
    for b, w in zip(bags, full):
        with torch.no_grad():
            b.weight.copy_(w)
    moments = [torch.zeros(t.num_rows, device="cuda") for t in specs]
    for it in range(2):
        lengths = rng.integers(0, 8, size=(len(specs), B))
        ids = torch.from_numpy(np.concatenate([rng.integers(0, t.num_rows, size=int(lengths[i].sum()))
                                               for i, t in enumerate(specs)])).cuda()
        dense = torch.from_numpy(rng.standard_normal((B, 13)).astype(np.float32)).cuda()
        labels = torch.from_numpy((rng.random(B) < 0.3).astype(np.float32)).cuda()
        got = m.step(lengths, ids, dense, labels)
        want = _reference_step(bottom, inter, top, bags, moments, lengths, ids, dense, labels, 0.05, 1e-8, 0.1)
        torch.cuda.synchronize()
        assert abs(float(got) - float(want)) <= 1e-5 * max(1.0, abs(float(want))), (it, float(got), float(want))
        for a, b in zip(list(m.bottom.parameters()) + list(m.top.parameters()),
                        list(bottom.parameters()) + list(top.parameters())):
            assert torch.allclose(a, b, rtol=1e-4, atol=1e-5), it
        for (s, w, mom), b, rmom in zip(m.emb.shard_tensors(0), bags, moments):
            assert torch.allclose(w, b.weight, rtol=1e-4, atol=1e-5), (it, s.table_id)
            assert torch.allclose(mom, rmom, rtol=1e-4, atol=1e-7), (it, s.table_id)
