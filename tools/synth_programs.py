"""Seeded synthetic MiniCUDA programs for differential sweeps (SURVEY.md 8(f)
rank 2: "acceptance-8-style differential sweeps ... on the corpus and
synthetic programs").

Templates follow the corpus access patterns: linear
thread index vs a size input with a grid of ceil(n / block); 2-D row * cols +
col; dynamic-shared partitions (sosfilt); per-thread local arrays filled in a
loop (kalman); static shared tiles; data-dependent atomics (push_node);
conditional frees (uaf).  Each knob (guard present / off by one, allocation
size +-1, cap values, block size) is drawn from a seeded RNG, so roughly a
third of the programs carry a bug.

    python tools/synth_programs.py N SEED   -> prints one JSON {name: source} dict
"""
from __future__ import annotations

import json
import random
import sys


def _caps(rng, names, lo=(0, 1), hi=(2, 12)):
    lines = []
    for n in names:
        lines.append(f"    assert({n} >= {rng.choice(lo)});")
        lines.append(f"    assert({n} <= {rng.randint(*hi)});")
    return "\n".join(lines)


def _pm(rng, p_bug=0.3):
    return rng.choice([" + 1", " - 1"]) if rng.random() < p_bug else ""


def t_linear(rng):
    blk = rng.choice((4, 8, 16, 32, 64))
    guard = rng.choice(["i < n", "i < n", "i <= n", "i < n + 1", None])
    off = _pm(rng)
    body = f"        a[i{off}] = 1;" if guard else f"    a[i{off}] = 1;"
    inner = (f"    if ({guard}) {{\n{body}\n    }}" if guard else body)
    return f"""__global__ void lin(int* a, int n) {{
    int i = threadIdx.x + blockIdx.x * blockDim.x;
{inner}
}}

void main() {{
    int n = __input();
{_caps(rng, ["n"])}
    int* a = cudaMalloc(n{_pm(rng, 0.2)});
    lin<<<(n + {blk - 1}) / {blk}, {blk}>>>(a, n);
}}
"""


def t_rowcol(rng):
    blk = rng.choice((4, 8, 16))
    guard = rng.choice(["c < cols", "c < cols", "c <= cols", None])
    off = _pm(rng, 0.25)
    st = f"m[r * cols + c{off}] = m[r * cols + c] + 1;"
    inner = f"    if ({guard}) {{\n        {st}\n    }}" if guard else f"    {st}"
    return f"""__global__ void rowcol(int* m, int rows, int cols) {{
    int r = blockIdx.x;
    int c = threadIdx.x;
{inner}
}}

void main() {{
    int rows = __input();
    int cols = __input();
{_caps(rng, ["rows", "cols"], lo=(1,), hi=(2, 8))}
    assert(cols <= {blk});
    int* m = cudaMalloc(rows * cols{_pm(rng, 0.2)});
    rowcol<<<rows, {blk}>>>(m, rows, cols);
}}
"""


def t_partition(rng):
    k = rng.choice((2, 3, 4))
    off = _pm(rng, 0.35)
    shm_extra = _pm(rng, 0.25)
    return f"""__global__ void parts(int* out, int s, int w) {{
    extern __shared__ int smem[];
    int* p0 = smem;
    int* p1 = &p0[s];
    int* p2 = &p0[s + s * w];
    int t = threadIdx.x;
    for (int i = 0; i < w; i++) {{
        p1[t * w + i{off}] = i;
    }}
    p2[t * {k}] = 1;
    out[t] = p0[t] + p1[t * w];
}}

void main() {{
    int s = __input();
    int w = __input();
{_caps(rng, ["s", "w"], lo=(1,), hi=(2, 8))}
    int* out = cudaMalloc(s);
    parts<<<1, s, s + s * w + s * {k}{shm_extra}>>>(out, s, w);
}}
"""


def t_loop_local(rng):
    extra = rng.choice(["", "", " + 1"])
    return f"""__global__ void loopy(int* src, int rd) {{
    int l_a[rd];
    for (int i = 0; i < rd{extra}; i++) {{
        l_a[i] = src[i];
    }}
    int j = rd - 1;
    src[j{_pm(rng, 0.2)}] = l_a[0];
}}

void main() {{
    int rd = __input();
{_caps(rng, ["rd"], lo=(1,), hi=(2, 10))}
    int* src = cudaMalloc(rd);
    loopy<<<1, 1>>>(src, rd);
}}
"""


def t_tile(rng):
    tile = rng.choice((8, 16, 32))
    blk = rng.choice((tile, tile, tile * 2, tile // 2))
    return f"""__global__ void tiled(int* out, int n) {{
    __shared__ int tile[{tile}];
    int i = threadIdx.x;
    tile[i] = i;
    if (i < n) {{
        out[i] = tile[i{_pm(rng, 0.3)}];
    }}
}}

void main() {{
    int n = __input();
{_caps(rng, ["n"], lo=(1,), hi=(2, 40))}
    int* out = cudaMalloc(n);
    tiled<<<1, {blk}>>>(out, n);
}}
"""


def t_atomic(rng):
    return f"""__global__ void push(int* nl, int* d1, int* d2, int nv, int deg) {{
    int i = threadIdx.x + blockIdx.x * blockDim.x;
    if (i < nv) {{
        for (int j = 0; j < deg; j++) {{
            int nb = nl[i * deg + j];
            atomicMin(&d1[nb], d2[i]);
        }}
    }}
}}

void main() {{
    int nv = __input();
    int deg = __input();
{_caps(rng, ["nv", "deg"], lo=(1,), hi=(2, 5))}
    int* nl = cudaMalloc(nv * deg);
    int* d1 = cudaMalloc(nv{_pm(rng, 0.2)});
    int* d2 = cudaMalloc(nv);
    nl[0] = __input();
    assert(nl[0] <= {rng.randint(2, 9)});
    push<<<(nv + 31) / 32, 32>>>(nl, d1, d2, nv, deg);
}}
"""


def t_uaf(rng):
    rel = rng.choice(("<", "<=", ">"))
    return f"""__global__ void use(int* data, int n) {{
    int i = threadIdx.x;
    if (i < n) {{
        data[i] = 2;
    }}
}}

void main() {{
    int flag = __input();
    int n = __input();
{_caps(rng, ["n"], lo=(1,), hi=(2, 8))}
    int* data = cudaMalloc(n);
    if (flag {rel} {rng.randint(0, 3)}) {{
        cudaFree(data);
    }}
    use<<<1, 8>>>(data, n);
}}
"""


TEMPLATES = (t_linear, t_rowcol, t_partition, t_loop_local, t_tile, t_atomic, t_uaf)


def generate(n: int, seed: int) -> dict:
    rng = random.Random(seed)
    out = {}
    for i in range(n):
        t = TEMPLATES[i % len(TEMPLATES)]
        out[f"synth/{i:04d}_{t.__name__[2:]}.mcu"] = t(rng)
    return out


if __name__ == "__main__":
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 70
    seed = int(sys.argv[2]) if len(sys.argv) > 2 else 2601215526
    print(json.dumps(generate(n, seed), indent=1))
