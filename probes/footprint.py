"""Memory-footprint analogue of the paper's max-batch claim:
expert weights of every MoE layer of a model resident in one B200's HBM, dense
bf16 vs the Samoyeds (1,2,32) device image (sizes from the library's own
smy_weight_layout), and the HBM left for everything else.  Host-only: the size
queries need no GPU.

    python probes/footprint.py > profiles/r1_footprint.md
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_10725_b200 as P  # noqa: E402

HBM = 180e9     # B200 (HBM3e)
# name: (hidden, ffn, routed experts, shared experts, MoE layers)
MODELS = {
    "Mixtral-8x7B": (4096, 14336, 8, 0, 32),
    "DeepSeek-MoE-16B": (2048, 1408, 64, 2, 27),       # layer 0 is dense in the released model
    "Qwen2-57B-A14B": (3584, 2560, 64, 8, 28),         # shared expert 20480 wide = 8 x 2560
}


def main():
    fmt = P.Format(1, 2, 32)
    print("# Expert-weight footprint per model, dense bf16 vs Samoyeds (1,2,32) on one B200\n")
    print("Sizes from `smy_weight_layout` (device image; the canonical values/codes/indices form is 0.578 B/elem).")
    print("'HBM left' = 180 GB minus all MoE layers' expert weights (attention, embeddings, KV cache not counted).\n")
    print("| model | MoE layers x experts | dense bf16 | (1,2,32) image | ratio | HBM left dense | HBM left (1,2,32) |")
    print("|---|---|---|---|---|---|---|")
    for name, (d, f, E, S, L) in MODELS.items():
        per_expert_dense = 3 * d * f * 2
        # the layout the layer holds: interleaved gate/up [2f x d] + down [d x f]
        img = P.weight_layout(2 * f, d, fmt)["image"] + P.weight_layout(d, f, fmt)["image"]
        n = L * (E + S)
        dense, comp = n * per_expert_dense, n * img
        print(f"| {name} | {L} x ({E}+{S}) | {dense / 1e9:.1f} GB | {comp / 1e9:.1f} GB | {dense / comp:.2f}x | "
              f"{(HBM - dense) / 1e9:.1f} GB | {(HBM - comp) / 1e9:.1f} GB |")


if __name__ == "__main__":
    main()
