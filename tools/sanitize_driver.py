"""Small-size driver for compute-sanitizer (tools/sanitize.sh): every libsg
kernel family once, at sizes the sanitizers finish in minutes.

    list ranking: rs_rank on random (ruling-set walk + binned records,
      refine, scatter, levels >= 1, cooperative top) and ordered lists
      (tile contraction), rs_rank_even (even splitters), wyllie_rank both
      variants;
    components: uf and sv, with and without the window partition
      (SG_CC_WBITS=12 forces several windows at small n), and the
      one-process multi-GPU entry (sg_cc_multi) on a one-device clique.
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1002_4482_b200 as g  # noqa: E402


def main():
    which = sys.argv[1] if len(sys.argv) > 1 else "all"
    dev = torch.device("cuda", 0)
    n = int(os.environ.get("SAN_N", 1 << 18))
    # inputs are generated on the host and copied in: initcheck tracks every
    # byte, and torch's device sort (the device generators) copies scratch
    # it never initialised
    if which in ("all", "list"):
        sl = g.SuccessorList(torch.from_numpy(g.gen_list(n, seed=1).succ).to(dev))
        r, st = g.rs_rank(sl, 1024)
        print("rs random", st.meta["path"], st.meta["levels"], st.meta["level_size"], int(r.max()),
              sorted({(x.kernel, x.blocks) for x in st.launch_log if x.kernel.startswith("rs4")}))
        # enough levels for the multi-CTA top (cooperative) at this size
        o = g.SuccessorList(torch.cat([torch.arange(1, n, device=dev), torch.tensor([n - 1], device=dev)]).to(torch.int32))
        r, st = g.rs_rank(o, 1024)
        print("rs ordered", st.meta["path"], int(r[0]))
        r, st = g.rs_rank_even(sl, 1024)  # sg_even_splitters
        print("rs even", st.meta["path"], len(st.meta["splitter_set"].splitter_node))
        r, _ = g.wyllie_rank(g.SuccessorList(torch.from_numpy(g.gen_list(1 << 14, seed=2).succ).to(dev)), 64)
        r, _ = g.wyllie_rank(g.SuccessorList(torch.from_numpy(g.gen_list(200, seed=3).succ).to(dev)), 128,
                             variant="single_block")
        print("wyllie ok")
    if which in ("all", "cc"):
        h = g.gen_random_graph(n, 8.0 * n / (n * (n - 1) // 2), seed=0)
        gr = g.EdgeGraph(n, torch.from_numpy(h.edges).to(dev))
        for variant in ("uf", "sv"):
            lab, st = g.sv_components(gr, 64, variant=variant)
            print("cc", variant, st.meta["rounds"], int(lab.max()))
        from paper_1002_4482_b200 import dist as sgdist
        lab, st = sgdist.sv_components_multi(gr, 64, devices=[0])  # sg_cc_multi (NCCL clique of one)
        print("cc multi", st.meta["rounds"], int(lab.max()))
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
