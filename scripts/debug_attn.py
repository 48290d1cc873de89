"""Dev script: decode-step logits vs oracle for several head dims / split settings (GPU)."""
import os, sys
import numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'baseline/_ref')
from paper_2602_00269_b200.config import tiny
from paper_2602_00269_b200.device import VoxDevice, Sampling
from oracle.llama import LlamaOracle
from oracle.workload import prompt_ids, request_seed
for name, cfg in [("hd64", tiny(max_slots=4, detok_enabled=False)),
                  ("hd128", tiny(max_slots=4, detok_enabled=False, n_heads=2, n_kv_heads=1, head_dim=128))]:
    for split in ("1", "4", ""):
        if split: os.environ["VOX_ATTN_SPLITS_TEST"] = split
        else: os.environ.pop("VOX_ATTN_SPLITS_TEST", None)
        dev = VoxDevice(cfg, 1234)
        orc = LlamaOracle(cfg, 1234)
        for P in (5, 21, 40):
            seed = request_seed(0, P)
            slot = dev.admit(seed, P, 40, Sampling(temperature=0.0))
            prompt = np.array(prompt_ids(seed, P, cfg.text_vocab))
            dev.forward(np.array([[slot, p, -1, 0] for p in range(P - 1)], np.int32), sample=False, sync=True, graph=False)
            orc.forward(P, prompt[:-1], np.arange(P - 1), want_logits=False)
            _, lg = dev.forward(np.array([[slot, P - 1, -1, 1]], np.int32), sample=False, full_logits=True, sync=True)
            ol, _ = orc.forward(P, prompt[-1:], np.array([P - 1]))
            k, v = dev.read_kv(0, slot, P // 2)
            print(name, "split", split or "auto", "P", P, "logit err %.4f" % np.abs(lg[0] - ol[0]).max(),
                  "k err %.4f v err %.4f" % (np.abs(k - orc.k[P][0, P // 2]).max(), np.abs(v - orc.v[P][0, P // 2]).max()), flush=True)
            dev.release(slot)
        dev.close()
