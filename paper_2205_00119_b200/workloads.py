"""The BASELINE.json workloads as plain data.

Pure Python on purpose: ``bench.py --impl reference`` and the CPU-side helpers
describe the same job without loading ``libmics.so`` (importing this module does
not import the package's native layer, see ``__init__.py``).
"""
from __future__ import annotations

from dataclasses import dataclass


def transformer_layer_params(hidden: int, intermediate: int, layers: int, vocab: int, seq_len: int) -> list:
    """Parameters per layer as the reference's derive_layers_from_transformer
    counts them (simulator.cpp:317-358): embedding (V + l) * h, then `layers`
    blocks of 4h^2 + 2h*i + 9h + i."""
    emb = (vocab + seq_len) * hidden
    block = 4 * hidden * hidden + 2 * hidden * intermediate + 9 * hidden + intermediate
    return [emb] + [block] * layers


@dataclass
class Workload:
    name: str
    layer_params: list
    p: int
    s: int
    grad_dtype: str = "f32"
    hier_k: int = 0
    n: int = 8
    micro_batch: int = 8          # samples per rank per micro-step
    note: str = ""
    hidden: int = 0               # step with compute: columns of X; layer l is W_l [E_l / hidden, hidden]
    seq_len: int = 1              # tokens per sample (X has micro_batch * seq_len rows)

    @property
    def tokens(self) -> int:
        return self.micro_batch * self.seq_len

    @property
    def params(self) -> int:
        return sum(self.layer_params)


def workloads() -> dict:
    """BASELINE.json configs."""
    bert_large = transformer_layer_params(1024, 4096, 24, 30522, 512)
    gpt2_xl = transformer_layer_params(1600, 6400, 48, 50257, 1024)
    bert_10b = transformer_layer_params(2560, 10240, 127, 32008, 512)
    return {
        "C1": Workload("C1 4-layer MLP H=1024 (W+b), n=8, p=2, s=4, fp32", [1024 * 1024 + 1024] * 4, p=2, s=4,
                       hidden=1024),
        "C3": Workload("C3 BERT-large-shaped 334M, n=8, p=2, s=4, fp32 grads", bert_large, p=2, s=4, hidden=1024,
                       seq_len=512),
        "C4": Workload("C4 GPT-2 1.5B-shaped, n=8, p=4, hierarchical k=2, bf16 grads", gpt2_xl, p=4, s=4,
                       grad_dtype="bf16", hier_k=2, hidden=1600, seq_len=1024),
        "C5p2": Workload("C5 10B dense (BERT-10B), n=8, p=2, bf16 grads", bert_10b, p=2, s=4, grad_dtype="bf16",
                         hidden=2560, seq_len=512),
        "C5p8": Workload("C5 10B dense (BERT-10B), n=8, p=8 (ZeRO-3), bf16 grads", bert_10b, p=8, s=4,
                         grad_dtype="bf16", hidden=2560, seq_len=512),
    }
