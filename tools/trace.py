"""Print the CTA-0 event trace written by VLASIM_TRACE=file (PROF builds).
python tools/trace.py file [u0 u1] [kernel-tag]   (default: the last kernel in the file)"""
import struct
import sys

NAMES = {36: "S0.item_start", 37: "S1.item_start", 38: "S0.unit_setup", 39: "S1.unit_setup", 1: "P.qload", 2: "P.kvload", 14: "M.bSdP_enter", 15: "M.bSdP_ready", 10: "M.pt_seen", 11: "M.dV+S2", 12: "M.ds_seen", 13: "M.dK+dP2", 
         20: "S0.s_seen", 21: "S1.s_seen", 22: "S0.pt_arr", 23: "S1.pt_arr", 24: "S0.dp_seen", 25: "S1.dp_seen",
         26: "S0.ds_arr", 27: "S1.ds_arr", 30: "E0.enter", 31: "E1.enter", 32: "E0.dkv_seen", 33: "E1.dkv_seen",
         34: "E0.done", 35: "E1.done", 50: "E.tmem_drained", 51: "E.dV_staged", 52: "E.dV_read",
         40: "M.ahead_adv", 41: "M.bnd_checked", 42: "M.next_unit", 43: "M.loads_seen"}
data = open(sys.argv[1], "rb").read()
off = 0
runs = []
while off < len(data):
    tag = data[off:off + 32].rstrip(b"\0").decode()
    n = struct.unpack_from("<Q", data, off + 32)[0]
    ev = struct.unpack_from(f"<{n}Q", data, off + 40)
    runs.append((tag, [(w >> 32, (w >> 16) & 0xFFFF, w & 0xFFFF) for w in ev]))
    off += 40 + 8 * n
want = sys.argv[4] if len(sys.argv) > 4 else runs[-1][0]
sel = [r for r in runs if r[0] == want][-4:]
tag = want
ev = sorted(e for r in sel for e in r[1])
if tag.startswith("k_bwd_dq"):
    NAMES = {1: "P.qdo_load", 10: "M.p_seen", 11: "M.dQ_iss", 12: "M.kv_seen", 13: "M.S+dP_iss", 20: "S.s_seen",
             21: "S.A_done", 22: "S.dp_seen", 23: "S.p_arr", 30: "E.enter", 31: "E.dq_seen", 32: "E.done"}
t0 = ev[0][0]
u0, u1 = (int(sys.argv[2]), int(sys.argv[3])) if len(sys.argv) > 3 else (100, 112)
print(tag, len(ev), "events; span", ev[-1][0] - t0, "cycles")
prev = None
for t, c, u in ev:
    if u0 <= u <= u1:
        d = "" if prev is None else f"+{t - prev}"
        print(f"{t - t0:10d} {d:>7s}  u={u:4d} {NAMES.get(c, c)}")
        prev = t
