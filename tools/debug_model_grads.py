import sys
sys.path.insert(0, ".")
import torch
from tests.test_gpu_model import _trainer, _oracle
tr = _trainer()
tokens = tr.synthetic_tokens().cuda()
losses = tr.forward_backward(tokens).cpu().double()
ref_losses, ref_grads, _ = _oracle(tr, tokens)
print(losses, ref_losses)
for (layer, tname), (dd, du) in ref_grads.items():
    for i in range(4):
        r = tr.meta.ranks[i]
        ga = tr.bank.block(tr.bank.G, layer, tname, "A", i)[:, :r].double().cpu()
        gb = tr.bank.block(tr.bank.G, layer, tname, "B", i)[:, :r].double().cpu().t()
        for nm, got, ref in (("A", ga, dd[i]), ("B", gb, du[i])):
            cos = (got * ref).sum() / (got.norm() * ref.norm() + 1e-30)
            print(layer, tname, i, nm, f"rel={((got-ref).norm()/ref.norm()).item():.3e} ratio={(got.norm()/ref.norm()).item():.3f} cos={cos.item():.4f}")
