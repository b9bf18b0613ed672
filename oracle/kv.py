"""Oracle: KV-cache byte model.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md §2.1 l.110: "the KV cache grows linearly with the sequence length and
model depth"; per-token bytes follow SPEC.md l.283-291:
    kv_bytes_per_token = 2 * layers * kv_heads * head_dim * bytes_per_element.
The shared prompt prefix holds P-1 tokens (reading R6); response KV lives in
pages of `page_tokens` tokens (R26).
"""


def kv_bytes_per_token(layers, kv_heads, head_dim, bytes_per_element=2):
    return 2 * layers * kv_heads * head_dim * bytes_per_element


def page_bytes(shape, page_tokens=16):
    return page_tokens * kv_bytes_per_token(shape.layers, shape.n_kv_heads, shape.head_dim)


def prefix_bytes(shape, prompt_len):
    return (prompt_len - 1) * kv_bytes_per_token(shape.layers, shape.n_kv_heads, shape.head_dim)


def peak_kv_bytes(shape, prompt_len, peak_pages, page_tokens=16):
    return prefix_bytes(shape, prompt_len) + peak_pages * page_bytes(shape, page_tokens)
