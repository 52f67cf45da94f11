"""Diagnostic: precision of one random token-loss case vs the oracle."""
import sys, numpy as np, torch
sys.path.insert(0, "."); sys.path.insert(0, "tests")
from test_token_loss_gpu import _case, _run_gpu
from oracle import grpo_oracle as O
from oracle.check import coeff_term_scale
from paper_2605_13276_b200 import grpo
for fused in (False, True):
    x, tokens, blp, rewards, ids = _case(2010, 4, 2, 3, 11, 8, torch.float32, spread=0.5, binary=False,
                                          ids=np.array([3, 1, 7, 5]))
    cfg = grpo.GrpoConfig(group_size=2, kl_coeff=0.2)
    loss, dl, st = _run_gpu(x, tokens, blp, rewards, ids, torch.float32, fused, cfg)
    oloss, odl, ost = O.grpo_token_grad(x, tokens, blp, rewards, ids, kl_coeff=0.2)
    e_tok = np.abs(st["lp_tok"].cpu().numpy().reshape(-1) - ost["lp_tok"])
    e_ch = np.abs(st["lp_chunk"].cpu().numpy() - ost["lp_chunk"])
    sc = coeff_term_scale(ost["lp_chunk"], blp, rewards, kl_coeff=0.2)
    e_co = np.abs(st["coeff"].cpu().numpy() - ost["coeff"]) / np.maximum(np.abs(ost["coeff"]), sc)
    print("fused", fused, "tok err max", e_tok.max(), "mean signed",
          float((st["lp_tok"].cpu().numpy().reshape(-1) - ost["lp_tok"]).mean()),
          "chunk err max", e_ch.max(), "coeff scaled err max", e_co.max())
