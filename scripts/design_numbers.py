"""Rewrite DESIGN.md's at-a-glance paragraph, §5.4 table and round-over-round sentence from a set of
bench lines in profiles/ (usage: design_numbers.py TAG, e.g. r2k; comparison lines stay r2e)."""
import json
import re
import sys

tag = sys.argv[1]


def L(n):
    return json.load(open(f"profiles/{n}.json"))


p = "DESIGN.md"
s = open(p).read()
d, g, g64, q = L(f"{tag}_llama3"), L(f"{tag}_gemma3_b512"), L(f"{tag}_gemma3_b64"), L(f"{tag}_qwen25")
b8, b2, r = L(f"{tag}_llama3_b8"), L(f"{tag}_llama3_b2"), L(f"{tag}_reference")
a = s.index("**At a glance (round 2")
b = s.index("## 1. The path and its boundary")
new = f"""**At a glance (round 2, one B200, `profiles/{tag}_*` — all lines from one box):** the Llama-3 drafter
head (V 128256, d 4096, M 256, B = 1, k = 32,32,8x6) runs one grid-wide launch per draft position —
{d['config']['us_per_draft_step']:.1f} us per step, {d['value']/1e3:.1f} k draft tokens/s (e2e through the public API with host copies: {d['e2e']['value']/1e3:.1f} k; the CPU
oracle: {d['cpu_baseline']['value']:.0f} tokens/s on 16 host cores, {d['cpu_baseline']['single_core']['value']:.1f} on one); roofline {d['roofline']['frac']:.2f} of the measured 6.55 TB/s for the
whole step (router included), 0.67 on the gathered cluster blocks while they stream; {d['config']['speedup_vs_dense']:.1f}x faster
than our own dense full-vocabulary head (1.05 GB at 6.5 TB/s) and ~16x faster than torch/cuBLAS.
The north-star targets (>= 0.70 of HBM for the step, >= 10.6x vs dense) are NOT met at B = 1 (§9
says what bounds it).  Batches run on a grouped cluster-major tcgen05 head (every selected cluster
block read once for all the rows that chose it) with the router's layer 1 on tcgen05: Gemma-3 at its
BASELINE batch of 512 requests takes {g['config']['us_per_draft_step']:.0f} us per step ({g['value']/1e3:.0f} k draft tokens/s, e2e {g['e2e']['value']/1e3:.0f} k, {g['roofline']['frac']:.2f} of the
HBM peak, {g['config']['speedup_vs_dense']:.1f}x vs our dense head, which itself beats cuBLAS {g['config']['dense_detail']['ours_k_eq_M_us']:.0f} vs {g['config']['dense_detail']['torch_cublas_us']:.0f} us; B = 64:
{g64['roofline']['frac']:.2f}).  Tree rows (Qwen, 10 rows per depth) run on a few-row one-launch router (§5.3e) and a
balanced tcgen05 tree head (§5.3d): {q['config']['us_per_draft_step']:.1f} us per step (90.6 at the start of this round's last session;
the CUDA-core fused step: 151.5 us), {q['config']['speedup_vs_dense']:.1f}x vs the best dense head; the same tree head in rows mode
serves Llama-3 B = 5-9 (B = 8: {b8['config']['us_per_draft_step']:.1f} us; the grouped head 105 us) and B = 2-3 run one grid step per
row (B = 2: {b2['config']['us_per_draft_step']:.1f} us, was 49).  All five BASELINE configs, the four SURVEY §8(f) NEXT rows and both
multi-GPU modes are built and parity-tested against the oracle (229 GPU tests, 43 CPU tests);
multi-GPU is exercised on CPU only (every GPU call here has one B200).  §5.4 has the table.

"""
s = s[:a] + new + s[b:]
s = re.sub(r"### 5\.4 Measured \(round 2, one B200, `profiles/r2[a-z]_\*\.json`",
           f"### 5.4 Measured (round 2, one B200, `profiles/{tag}_*.json`", s)
a = s.index("| Config (BASELINE.json) | Path (dominant kernel) | us / draft step |")
b = s.index("(e2e: the public API with host copies;")


def row(cfg, path, n, dense_note=None):
    x = L(n)
    c = x["config"]
    dd = c["dense_detail"]
    dn = dense_note or f"{dd['best_us']:.0f}"
    return (f"| {cfg} | {path} | {c['us_per_draft_step']:.1f} | {x['value']/1e3:.1f} k ({x['e2e']['value']/1e3:.1f} k) | "
            f"{x['roofline']['frac']:.2f} | {dn} | {c['speedup_vs_dense']:.1f}x |")


t = ["| Config (BASELINE.json) | Path (dominant kernel) | us / draft step | draft tokens/s (e2e) | frac | dense us | speedup vs dense |",
     "|---|---|---|---|---|---|---|"]
dd = d["config"]["dense_detail"]
t.append(row("Llama-3 (V 128256, d 4096, M 256), B = 1, k 32,32,8x6", "grid step `gstep_kernel`", f"{tag}_llama3",
             f"{dd['ours_k_eq_M_us']:.1f} (ours) / {dd['torch_cublas_us']:.0f} (cuBLAS)"))
t.append(row("Llama-3, B = 2", "one grid step per row `gstep_kernel`", f"{tag}_llama3_b2"))
t.append(row("Llama-3, B = 4", "fused multi-row step `step_kernel`", f"{tag}_llama3_b4"))
t.append(row("Llama-3, B = 6", "few-row router + tree head, rows mode `th_kernel`", f"{tag}_llama3_b6"))
t.append(row("Llama-3, B = 8", "few-row router + tree head, rows mode `th_kernel`", f"{tag}_llama3_b8"))
t.append(row("Llama-3, B = 8 (`DS_TH_ROWS=0`, earlier box)", "grouped tcgen05 head `gh_head_kernel`", "r2e_llama3_b8_gh"))
for B in (16, 32, 64):
    t.append(row(f"Llama-3, B = {B}", "grouped tcgen05 head `gh_head_kernel`", f"{tag}_llama3_b{B}"))
t.append(row("Tiny (V 32000, d 1024, M 64), B = 1, k = 8", "grid step", f"{tag}_tiny"))
t.append(row("Llama-2 (V 32000, d 4096, M 128), B = 1, k 16->4", "grid step", f"{tag}_llama2"))
t.append(row("Qwen-2.5 (V 151936, d 3584), tree 10 rows / depth", "few-row router + balanced tree head `th_kernel`",
             f"{tag}_qwen25"))
t.append(row("Qwen-2.5 tree (`DS_TH=0 DS_META_ROWS=0`, earlier box)", "split-K router + general `tc_head_kernel`",
             "r2e_qwen25_tchead"))
t.append(row("Qwen-2.5 tree (`DS_DISABLE_TC=1`, earlier box)", "CUDA-core fused step `step_kernel`", "r2e_qwen25_cudacore"))
dd = g["config"]["dense_detail"]
t.append(row("Gemma-3 (V 262144, d 5376, M 512), B = 512", "router (tcgen05 layer 1) + grouped `gh_head_kernel`",
             f"{tag}_gemma3_b512", f"{dd['ours_k_eq_M_us']:.0f} (ours) / {dd['torch_cublas_us']:.0f} (cuBLAS)"))
dd = g64["config"]["dense_detail"]
t.append(row("Gemma-3, B = 64 (round 1: 559 us, 0.58)", "router + grouped `gh_head_kernel`", f"{tag}_gemma3_b64",
             f"{dd['ours_k_eq_M_us']:.0f} (ours) / {dd['torch_cublas_us']:.0f} (cuBLAS)"))
s = s[:a] + "\n".join(t) + "\n\n" + s[b:]
b64 = L(f"{tag}_llama3_b64")
a = s.index("Round 1 -> round 2 on the same workloads:")
e = s.index("The dense comparator (our k = M head at B = 1", a)
s = s[:a] + f"""Round 1 -> round 2 on the same workloads: Llama-3 B = 1 22.3 -> {d['config']['us_per_draft_step']:.1f} us; Gemma-3 at its BASELINE batch
(B = 512; round 1 only measured B = 64, 559 us) 20984 us (round-1 code at B = 512) -> {g['config']['us_per_draft_step']:.0f} us; Gemma-3 B = 64
559 -> {g64['config']['us_per_draft_step']:.0f} us; Llama-3 B = 64 326 -> {b64['config']['us_per_draft_step']:.0f} us; Qwen tree 89.7 -> {q['config']['us_per_draft_step']:.1f} us.  e2e: the tree configs'
e2e leg draws the same sibling rows as the timed workload (it drew independent rows: a 2x larger
union), and three copy schedules are timed with the fastest reported (one H2D copy per cycle;
position 0 first and the rest behind step 0; per-position copies overlapping the previous step):
Gemma-3 B = 512 e2e 603 k -> {g['e2e']['value']/1e3:.0f} k tokens/s.  CPU oracle on the same Llama-3 workload (same k-means
partition): {d['cpu_baseline']['value']:.1f} draft tokens/s on 16 host threads, {d['cpu_baseline']['single_core']['value']:.1f} on one core (`cpu_baseline.single_core`);
`--impl reference`: {r['value']:.1f}.  North-star target "beats a dense head by >= |V| / (|V_S| + M) x 0.6": mean
|V_S| = 6988 gives 10.6x; measured {d['config']['speedup_vs_dense']:.1f}x (ours) / {d['config']['dense_detail']['torch_cublas_us']/d['config']['us_per_draft_step']:.1f}x (cuBLAS).  """ + s[e:]
s = re.sub(r"Tree rows \(Qwen, §5\.3d-e\): 90\.6 -> [0-9.]+ us per step",
           f"Tree rows (Qwen, §5.3d-e): 90.6 -> {q['config']['us_per_draft_step']:.1f} us per step", s)
s = re.sub(r"Gemma-3 B = 64 runs at [0-9.]+ of the copy peak \(round 1: 0\.58\); B = 512 at [0-9.]+ of",
           f"Gemma-3 B = 64 runs at {g64['roofline']['frac']:.2f} of the copy peak (round 1: 0.58); B = 512 at {g['roofline']['frac']:.2f} of", s)
open(p, "w").write(s)
print("ok")
