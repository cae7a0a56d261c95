"""Summarise gpurun_out/tab67.jsonl (tools/tab67_sweep.sh) as the paper's Tab. 6/7 layout: whole-context
prefill latency (s) and decode latency (s/token) per head-group granularity, next to the paper's RTX 4090
HeadInfer rows (Llama-3-8B whole model; ours is the attention path on one B200).

    python tools/tab67_table.py gpurun_out/tab67.jsonl > profiles/tab67_b200_r01.md
"""
import json
import sys

CTX = [1024, 10240, 102400, 409600, 1048576]
CTX_LABEL = ["1K", "10K", "100K", "400K", "1M"]
# paper, HeadInfer rows of Tab. 6 (prefill s) and Tab. 7 (decode s/token) at 1K, 10K, 100K, 400K, 1M;
# the paper's "head=h/group=n" means n groups of h kv heads, i.e. our G = h
PAPER = {
    8: ("head=8/group=1", [0.12, 1.24, 30.2, 357, None], [0.03, 0.09, 0.66, 2.58, None]),
    4: ("head=4/group=2", [0.13, 1.23, 30.2, 351, 2033], [0.04, 0.10, 0.67, 2.58, 6.41]),
    2: ("head=2/group=4", [0.14, 1.23, 30.5, 353, 2035], [0.06, 0.11, 0.68, 2.59, 6.46]),
    1: ("head=1/group=8", [0.21, 1.27, 31.2, 356, 2054], [0.10, 0.14, 0.71, 2.61, 6.51]),
    -2: ("Adaptive", [0.13, 1.24, 30.2, 351, 2033], [0.03, 0.09, 0.66, 3.03, 6.41]),
}


def fmt(v, nd=3):
    return "-" if v is None else (f"{v:.{nd}g}" if v < 100 else f"{v:.0f}")


def main(path):
    runs = {}
    for ln in open(path):
        ln = ln.strip()
        if ln:
            r = json.loads(ln)
            runs[(r["head_group_arg"], r["context"])] = r
    print("# Tab. 6/7 on one B200 (tools/tab67_sweep.sh): whole-context prefill (s) and decode (s/token), "
          "Llama-3-8B attention shapes, attention path only, chunk 18944, one-head staging ring")
    print("# paper values: HeadInfer on one RTX 4090, whole model, chunk 10K (P:L568-606)\n")
    for title, key, pidx in (("Prefill latency (s)", "prefill_s", 1), ("Decode latency (s/token)", "decode_ms_per_token", 2)):
        print(f"## {title}\n")
        print("| G (kv heads per unit) | " + " | ".join(CTX_LABEL) + " |")
        print("|---|" + "---|" * len(CTX))
        for g in (8, 4, 2, 1, -2):
            cells = []
            for c, p in zip(CTX, PAPER[g][pidx]):
                r = runs.get((g, c))
                v = None if r is None else (r[key] / 1e3 if key == "decode_ms_per_token" else r[key])
                cells.append(f"{fmt(v)} ({fmt(p)})")
            name = {-2: "paper's adaptive schedule"}.get(g, str(g))
            print(f"| {name} [paper: {PAPER[g][0]}] | " + " | ".join(cells) + " |")
        print("\nours (paper)\n")


if __name__ == "__main__":
    main(sys.argv[1])
