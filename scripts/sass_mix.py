"""Static SASS instruction-class counts per kernel family of libqeft_b200.so (cuobjdump -sass):
the evidence that the hot kernels use tcgen05 (UTC*MMA, LDTM), TMA / bulk copies (UTMALDG,
UBLKCP) and what else they issue. Writes a markdown table to stdout."""
import collections, re, subprocess, sys

so = sys.argv[1] if len(sys.argv) > 1 else "paper_2410_08661_b200/libqeft_b200.so"
txt = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
fams = collections.OrderedDict()
cur = None
for line in txt.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        name = m.group(1)
        fam = re.sub(r"^_ZN\d+_GLOBAL__N__\w+?_\d+(\w+?)E.*", r"\1", name)
        mm = re.search(r"(gemv2_kernel|gemv_kernel|gemm_kernel|wgrad_kernel|adam_step_kernel|adam_kernel|sqnorm_partial|"
                       r"shadow_kernel|grid_kernel|optq_\w+_kernel|rtn_kernel|rmsnorm_\w+|rope\w*kernel|silu_mul_\w+|"
                       r"ref_to_tiles_kernel|tiles_to_ref_kernel|pack_\w+_kernel|gather_cols_kernel|dequant_full_kernel)", name)
        cur = mm.group(1) if mm else "other"
        fams.setdefault(cur, collections.Counter())
        fams[cur]["#instantiations"] += 1
        continue
    m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_]+)", line)
    if m and cur:
        fams[cur][m.group(1)] += 1
key = ["UTCHMMA", "UTCQMMA", "UTCBAR", "LDTM", "STTM", "UTMALDG", "UTMASTG", "UBLKCP", "HMMA", "LDGSTS",
       "LDS", "STS", "LDG", "STG", "LOP3", "SHF", "FFMA", "FADD", "IMAD", "BRA", "SYNCS"]
print("| kernel family | instantiations | " + " | ".join(key) + " |")
print("|---|---|" + "---|" * len(key))
for fam, c in fams.items():
    if fam == "other":
        continue
    print(f"| `{fam}` | {c['#instantiations']} | " + " | ".join(str(sum(v for k, v in c.items() if k == kk))
                                                                for kk in key) + " |")
