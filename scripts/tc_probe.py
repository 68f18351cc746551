import ctypes as C, sys
sys.path.insert(0, "/root/repo")
from paper_2505_01572_b200 import abi
L = abi.test_lib()
L.ps_test_tc_probe.argtypes = [C.c_int32, C.c_int32, C.c_int32, C.POINTER(C.c_double)]
MODES = [(0, "cp 16KB"), (1, "8 MMA A=tmem"), (2, "8 MMA A=smem"), (3, "cp + 8 MMA tmem"),
         (4, "4 MMA N32 1acc"), (5, "8 MMA N16 2acc"), (6, "4 MMA N32 2acc"), (7, "4 MMA N16 1acc"),
         (8, "8 MMA N16 4acc"), (9, "4 MMA N32 4acc"), (10, "W as B N256 32KB"), (11, "W as B N128 16KB"),
         (12, "TMEM->smem 256 col"), (13, "TMEM->regs 256 col")]
ns = C.c_double()
abi.test_check(L.ps_test_tc_probe(2, 200000, 4, C.byref(ns)))     # warm up the clocks
for mode, name in MODES[int(sys.argv[1]) if len(sys.argv) > 1 else 0:]:
    for depth in (4,):
        ns = C.c_double()
        abi.test_check(L.ps_test_tc_probe(mode, 50000, depth, C.byref(ns)))
        print(f"{name:18s} depth {depth:2d}: {ns.value:8.1f} ns/unit", flush=True)

ns = C.c_double()
abi.test_check(L.ps_test_tc_probe2(50000, 4, C.byref(ns)))
print(f"{'2-CTA M256 N32 4 MMA':18s} depth  4: {ns.value:8.1f} ns/unit (16 KB per SM)", flush=True)

# mma.sync (legacy HMMA path, used by the decode attention): issue interval
for warps in (1, 4):
    for chains in (1, 2, 4, 8):
        ns, cyc = C.c_double(), C.c_double()
        abi.test_check(L.ps_test_hmma_probe(warps, chains, 20000, C.byref(ns), C.byref(cyc)))
        print(f"HMMA m16n8k16 warps {warps} chains {chains}: {ns.value:6.2f} ns, {cyc.value:6.2f} cycles per HMMA per warp",
              flush=True)
