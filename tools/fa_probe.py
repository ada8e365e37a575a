import torch, time
q = torch.randn(4096, 32, 128, dtype=torch.bfloat16, device="cuda")
k = torch.randn(4096, 8, 128, dtype=torch.bfloat16, device="cuda")
v = torch.randn(4096, 8, 128, dtype=torch.bfloat16, device="cuda")
cu = torch.tensor([0, 1000, 4096], dtype=torch.int32, device="cuda")
for name in ("flash_attn", "vllm_fa", "flashinfer", "sdpa"):
    try:
        if name == "flash_attn":
            from flash_attn import flash_attn_varlen_func
            o = flash_attn_varlen_func(q, k, v, cu, cu, 3096, 3096, causal=True)
        elif name == "vllm_fa":
            from vllm.vllm_flash_attn import flash_attn_varlen_func as f2
            o = f2(q, k, v, max_seqlen_q=3096, cu_seqlens_q=cu, max_seqlen_k=3096, cu_seqlens_k=cu, causal=True)
        elif name == "flashinfer":
            import flashinfer
            ws = torch.empty(128 << 20, dtype=torch.uint8, device="cuda")
            w = flashinfer.BatchPrefillWithRaggedKVCacheWrapper(ws, "NHD")
            w.plan(cu, cu, 32, 8, 128, causal=True)
            o = w.run(q, k, v)
        else:
            o = torch.nn.functional.scaled_dot_product_attention(q[:1000].transpose(0,1), k[:1000].repeat_interleave(4,1).transpose(0,1), v[:1000].repeat_interleave(4,1).transpose(0,1), is_causal=True)
        torch.cuda.synchronize()
        print(name, "OK", tuple(o.shape) if hasattr(o, "shape") else type(o))
    except Exception as e:
        print(name, "FAIL", type(e).__name__, str(e)[:200])
