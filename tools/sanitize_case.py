"""One small invocation of every entry point of the hot path (for compute-sanitizer).

    compute-sanitizer --tool {memcheck,racecheck,synccheck} python tools/sanitize_case.py <case>

cases: tiny (fp32 SIMT), n512_d64 (bf16 split-group fused + tcgen05 unfused), n512_d128 (paired
fused), st_d128 (residue decomposition, two passes), str_d64 (permuted plain STRIDED)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2407_16847_b200 import splat as S  # noqa: E402
from workloads import CONFIG_BY_NAME, Config, Pattern, make_qkv  # noqa: E402

CASES = {
    "tiny": CONFIG_BY_NAME["tiny"],
    "n512_d64": Config("n512_d64", Pattern("global_local", 512, lo=64, hi=64, n_global=8), 1, 2, 64, "bf16", 601),
    "n512_d128": Config("n512_d128", Pattern("window", 512, lo=100, hi=30), 1, 2, 128, "bf16", 602),
    "st_d128": Config("st_d128", Pattern("strided_local", 1024, stride=16, causal=1), 1, 2, 128, "bf16", 603),
    "str_d64": Config("str_d64", Pattern("strided", 1024, stride=16), 1, 2, 64, "bf16", 604),
}
cfg = CASES[sys.argv[1]]
q, k, v = make_qkv(cfg)
Q, K, V = q.cuda(), k.cuda(), v.cuda()
a = S.Acsr(cfg.pattern)
B, H = cfg.B, cfg.H
Sd = torch.empty(B * H * a.nnz, dtype=torch.float32, device="cuda")
Pd = torch.empty(B * H * a.nnz, dtype=cfg.torch_dtype, device="cuda")
O = torch.empty_like(Q)
for _ in range(2):
    S.splat_sparse_mhsa(a, Q, K, V, O, cfg.scale)
    S.splat_rsddmm(a, Q, K, Sd, cfg.scale)
    S.splat_sparse_softmax(a, Sd, Pd, B, H)
    S.splat_rspmm(a, Pd, V, O)
torch.cuda.synchronize()
print(cfg.name, "ok", float(O.float().abs().sum()))
