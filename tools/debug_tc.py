import sys, numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from test_gpu_decode_tc import build
from paper_2506_07311_b200 import AttentionConfig, MaskMeta, paged_attention, gathered_attention
lengths = [40, 130, 7]
pool, store, keys, vals = build(lengths, 2, 128, 16, torch.bfloat16)
cfg = AttentionConfig(head_count=8, head_dim=128, page_size=16, kv_head_count=2)
view = store.batch_view(list(range(3)))
for name, meta in (("self", MaskMeta.self_attention(view)), ("suffix", MaskMeta.suffix(view, [3, 1, 7])), ("decode", MaskMeta.decode(view))):
    torch.manual_seed(0)
    q = torch.randn((meta.query_count, 8, 128), device="cuda").bfloat16()
    a = paged_attention(q, store, meta, cfg)
    b = paged_attention(q, store, meta, cfg)
    gk, gv = store.gather_view(view)
    c = gathered_attention(q, gk, gv, meta, cfg)
    d = (a - c).abs()
    idx = torch.nonzero(d.amax(dim=(1, 2)) > 0).flatten().tolist()
    print(name, "run-to-run equal", torch.equal(a, b), "paged==gathered", torch.equal(a, c), "maxdiff", d.max().item(), "queries differing", idx[:20], len(idx))
    print("  q_seq/q_pos of differing", [(int(meta.q_seq[i]), int(meta.q_pos[i])) for i in idx[:10]])
    print("  gk equal to cache rows", torch.equal(gk, store.keys[torch.from_numpy(store.view_row_indices(view)).cuda()]))
