"""Build the ablation variants of libpfac into paper_1811_10498_b200/_lib/alt/.

Each variant is the product library with one PFAC_* knob flipped; scripts/ablations.sh benches them.
"""
import concurrent.futures as cf
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1811_10498_b200 import _build  # noqa: E402

ALT = os.path.join(os.path.dirname(_build.LIB), "alt")
VARIANTS = {
    "text_direct": ["PFAC_TEXT_DIRECT=1"],   # text read from global (L1/L2), no TMA staging
    "window0": ["PFAC_WINDOW_MAX=0"],        # no transition-table rows in shared memory
    "jtable": ["PFAC_FB16=0"],               # uint16 images: 4^8 jump table instead of filter + J2
    "nopersist": ["PFAC_NO_PERSIST"],        # no L2 access-policy window over J2
    "merged_f": ["PFAC_MERGED_F=1"],         # the paper's merged array: F(s) inside each T row
    "tab_cg": ["PFAC_TAB_CG=1"],             # table loads ld.global.cg (L2 only), the paper's -dlcm=cg
    "push_ballot": ["PFAC_PUSH_SCAN=0"],     # A/B: the round-1 queue push (one ballot round per position)
    "nolog": ["PFAC_MATCH_LOG=0"],           # A/B: no match log (dense matches spill to the out[] re-read)
    "nolog_ballot": ["PFAC_MATCH_LOG=0", "PFAC_PUSH_SCAN=0"],
    "ipl2": ["PFAC_DRAIN_IPL=2"],            # A/B: two queued positions per lane per drain round (2048-position slices too)
    "ipl1": ["PFAC_DRAIN_IPL_1K=1"],
    "ipl3": ["PFAC_DRAIN_IPL_1K=3"],
    "ipl4": ["PFAC_DRAIN_IPL_1K=4"],         # A/B: one per lane in the 1024-position-slice kernels too
    "nofstep": ["PFAC_FSTEP=0"],             # A/B: no FSTEP flag in uint16 chain rows
    "k2max10": ["PFAC_K2MAX=10"],            # A/B: second-level jump over 10-mers at most (4 MiB J2; cfg4 takes 11)
    "defer": ["PFAC_DEFER=1"],               # A/B: a group's last drain round resolved after the next group's filter step
    "chain16": ["PFAC_CHAIN32=0"],           # A/B: 16 forced bases per uint32 chain row (round 1)
    "noend": ["PFAC_ENDDEAD=0"],             # A/B: no end-state answers in uint32 chain rows
    "fb_add": ["PFAC_FB_LOP=0"],             # A/B: filter word addresses as base + offset (one more IADD per lookup)
    "jpre_probe": ["PFAC_JPRE=1", "PFAC_JPRE_PROBE=1"],     # probe: the J2 prefetch buffer allocated (shared memory), not used
    "jpre4": ["PFAC_JPRE=1", "PFAC_JPRE_K=4"],              # A/B: 4 J2 prefetch slots per lane
    "jpre": ["PFAC_JPRE=1"],                 # A/B: J2 prefetch (cp.async at filter time) in the 1024-position uint32 text kernels
    "j2na": ["PFAC_J2_NA=1"],                # A/B: J2 and HR loads ld.global.nc.L1::no_allocate
    "tabna": ["PFAC_TAB_NA=1"],              # A/B: every table load L1::no_allocate
    "mt1k": ["PFAC_MT_1K=1024"],             # A/B: 32 warps per CTA in the 1024-position-slice text kernels
    "mt1k960": ["PFAC_MT_1K=960"],           # A/B: 30 warps per CTA (shared memory stays under the 196-KB carve-out on cfg4)
    "mt1k_q96": ["PFAC_MT_1K=1024", "PFAC_QEXTRA_1K=96"],  # A/B: 32 warps with a shorter queue (cfg4: under 196 KB)
    "j2a32": ["PFAC_J2_NA32=0"],             # A/B: J2 / HR loads of uint32 images L1-allocating
    "nolds": ["PFAC_LDS_ADDR=0"],            # A/B: shared-window addresses from generic pointers (S2R per conversion)
    "win1600": ["PFAC_WINDOW_MAX=1600"],     # A/B: at most 1600 rows in shared memory (cfg5: a smaller carve-out, more L1)
    "w32ipl1": ["PFAC_QEXTRA_1K=128", "PFAC_DRAIN_IPL_1K=1"],  # A/B: 32 warps, 1 drain item per lane (same queue)
    "w32ipl3": ["PFAC_MT_1K=1024", "PFAC_QEXTRA_1K=64", "PFAC_DRAIN_IPL_1K=3"],  # A/B: 32 warps, 3 drain items per lane
    "w32ipl4": ["PFAC_MT_1K=1024", "PFAC_QEXTRA_1K=32", "PFAC_DRAIN_IPL_1K=4"],  # A/B: 32 warps, 4 drain items per lane
    "w28q96": ["PFAC_QEXTRA_1K=96"],         # A/B: 28 warps with the shorter queue (isolates the queue length)
    "mt1k640": ["PFAC_MT_1K=640"],           # A/B: 20 warps per CTA in the 1024-position-slice text kernels
    "mt1k512": ["PFAC_MT_1K=512"],           # A/B: 16 warps per CTA (shared memory under the 164-KB carve-out: more L1)
    "nojpre": ["PFAC_JPRE=0"],               # A/B: no J2 prefetch (cp.async at filter time) in the 1024-position uint32 text kernels
}

if __name__ == "__main__":
    os.makedirs(ALT, exist_ok=True)
    names = sys.argv[1:] or list(VARIANTS)
    with cf.ThreadPoolExecutor(4) as ex:
        futs = {ex.submit(_build.build, out=os.path.join(ALT, f"libpfac_{n}.so"), defines=VARIANTS[n]): n
                for n in names}
        for f in cf.as_completed(futs):
            print(futs[f], "->", f.result())
