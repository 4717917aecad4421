"""SASS opcode mix of the hot kernels in libtsg.so (cuobjdump -sass): counts of
the FP64 tensor (DMMA), FP64 FMA (DFMA/DADD/DMUL), bulk-copy / TMA (UBLKCP,
UTMALDG), mbarrier (SYNCS), barrier (BAR), shuffle, shared / global load-store
and MUFU instructions per kernel.   python tools/sass_mix.py > profiles/r02/sass_opcode_mix.txt"""
import collections, os, re, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2308_16395_b200", "libtsg.so")
HOT = ["proj0_colsr_kernel", "proj0_cols_kernel", "proj0_tma_kernel", "proj_dmma_kernel", "tail_kernel",
       "isvd_clu_kernel", "isvd_grid_kernel", "isvd_cta_kernel", "gram_partial_dmma_kernel",
       "gram_partial_narrow_kernel", "tridiag_coop_kernel", "tri_bisect_kernel", "tri_invit_kernel",
       "tri_backtransform_kernel", "sym_eig_coop_kernel", "isvd_update_kernel", "isvd_inner_kernel",
       "pgram_kernel", "recon"]
GROUPS = [("DMMA", r"^DMMA"), ("DFMA/DADD/DMUL", r"^(DFMA|DADD|DMUL)"), ("UBLKCP", r"^UBLKCP"),
          ("UTMA*", r"^UTMA"), ("SYNCS", r"^SYNCS"), ("BAR", r"^BAR"), ("SHFL", r"^SHFL"),
          ("LDS", r"^LDS"), ("STS", r"^STS"), ("LDG", r"^LDG"), ("STG", r"^STG"),
          ("LDL/STL", r"^(LDL|STL)"), ("MUFU", r"^MUFU"), ("CCTL/FENCE", r"^(CCTL|MEMBAR|FENCE|ERRBAR)")]
out = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
kern, counts = None, collections.OrderedDict()
for line in out.splitlines():
    m = re.match(r"\s*Function : (\S+)", line)
    if m:
        name = subprocess.run(["c++filt", m.group(1)], capture_output=True, text=True).stdout.strip()
        kern = name if any(h in name for h in HOT) else None
        if kern:
            counts[kern] = collections.Counter()
        continue
    if kern:
        m = re.match(r"\s*/\*[0-9a-f]+\*/\s+(?:@!?U?P\d+\s+)?([A-Z0-9_.]+)", line)
        if m:
            op = m.group(1)
            counts[kern]["total"] += 1
            for g, rx in GROUPS:
                if re.match(rx, op):
                    counts[kern][g] += 1
print("SASS opcode mix, libtsg.so (sm_100a), static instruction counts per kernel")
hdr = ["total"] + [g for g, _ in GROUPS]
print("kernel".ljust(70) + " ".join(h[:8].rjust(8) for h in hdr))
for k, c in counts.items():
    short = k.replace("(anonymous namespace)::", "").replace("tsg::", "").replace("<unnamed>::", "")
    short = re.sub(r"\(.*", "", short).replace("void ", "")
    print(short[:69].ljust(70) + " ".join(str(c.get(h, 0)).rjust(8) for h in hdr))
