"""Diagnostic: where do device and oracle logits diverge (tiny config)?"""
import sys
import numpy as np
sys.path.insert(0, ".")
from oracle.llama import LlamaOracle
from oracle.workload import prompt_ids, request_seed
from oracle.weights import bf16_round
from paper_2602_00269_b200.config import tiny
from paper_2602_00269_b200.device import Sampling, VoxDevice

cfg = tiny()
dev = VoxDevice(cfg, weight_seed=1234)
orc = LlamaOracle(cfg, 1234)
P = 21
seed = request_seed(0, 7)
slot = dev.admit(seed, P, 40, Sampling(temperature=0.0, repetition_penalty=1.3))
prompt = np.array(prompt_ids(seed, P, cfg.text_vocab))
dev.forward(np.array([[slot, p, -1, 0] for p in range(P - 1)], np.int32), sample=False, sync=True, graph=False)
orc.forward("r", prompt[:-1], np.arange(P - 1), want_logits=False)
for L in range(cfg.n_layers):
    for pos in (0, 1, P // 2, P - 2):
        k, v = dev.read_kv(L, slot, pos)
        ok, ov = orc.k["r"][L, pos], orc.v["r"][L, pos]
        print(f"layer {L} pos {pos}: K diff frac {np.mean(k != ok):.4f} max {np.abs(k-ok).max():.3e} |k| {np.abs(ok).max():.2f};"
              f" V diff frac {np.mean(v != ov):.4f} max {np.abs(v-ov).max():.3e}")
for step in range(4):
    _, lg = dev.forward(np.array([[slot, P - 1 + step, -1 if step == 0 else 128300, 1]], np.int32), sample=False,
                        full_logits=True, sync=True)
    tok = prompt[-1:] if step == 0 else np.array([128300])
    ol, x = orc.forward("r", tok, np.array([P - 1 + step]))
    d = lg[0].astype(np.float64) - ol[0]
    print(f"step {step}: logits std {ol[0].std():.3f} max|d| {np.abs(d).max():.3e} rms d {np.sqrt((d*d).mean()):.3e}")
