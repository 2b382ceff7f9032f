"""Memory formulas of §3.1 (oracle; test infrastructure only).

Eq. 1: Memory_KV = 2*h*b*k*x*p, x = m*n.  The printed product omits
the head dim d although d is defined in the same sentence; SPEC.md S:111 and
reading Q14 restore it: 2 * layers * b * kv_heads * d_head * x * p.  The build
also reserves N tree-scratch slots per sequence (reading Q14).

Eq. 3: Memory_buffers = b*N*w + b*S*l*w + b*S*l*l*w (elements; times p
bytes per Eq. 6).

Eq. 4: Memory_heads = 0.6 GB * l; a Medusa-1 head has d*d + d + V*d
parameters (reading Q6).
"""


def kv_bytes(n_layers, batch, n_kv_heads, head_dim, seq_len, bytes_per=2, tree_nodes=0):
    return 2 * n_layers * batch * n_kv_heads * head_dim * (seq_len + tree_nodes) * bytes_per


def kv_bytes_per_token(n_layers, n_kv_heads, head_dim, bytes_per=2):
    return kv_bytes(n_layers, 1, n_kv_heads, head_dim, 1, bytes_per)


def buffer_bytes(N, S, l, vocab, batch=1, bytes_per=2):
    return (batch * N * vocab + batch * S * l * vocab + batch * S * l * l * vocab) * bytes_per


def medusa_head_params(d_model, vocab):
    return d_model * d_model + d_model + vocab * d_model
