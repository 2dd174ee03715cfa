"""Render CTA 0's barrier-wait timeline written by JG_WAIT_PROF=2 (gpurun_out/trace_<tag>.txt).

    python tools/trace_view.py gpurun_out/trace_bwd.txt [first_item] [n_items]
    python tools/trace_view.py gpurun_out/trace_fwd.txt [first_item] [n_items]   (forward kernel names)

Each line: time in cycles since the first event, role column, event. A wait prints as
"name ... +cycles" at its exit. Items are delimited by the producer's K/V issue (code 50).
"""
import sys

NAMES = {0: "P.k_empty", 1: "P.qd_empty", 2: "P.v_empty", 3: "P.item_empty", 8: "S.k_full", 9: "S.v_full",
         10: "S.qd_full", 11: "S.pt_free", 12: "S.dq_empty", 16: "X.qd_full", 17: "X.st_full", 18: "X.pds_empty",
         24: "D.dq_full", 25: "D.stage_bar", 26: "D.dkv_full", 33: "G.dkv_empty", 37: "G.p_full",
         50: "P.KV-issued", 56: "S.start", 57: "S.S-issued", 58: "S.commit-st", 82: "G.commit-all", 83: "G.start", 84: "G.dq-issued", 85: "G.dv-issued", 66: "X.p_full-arrive",
         74: "D.dkv-done", 75: "D.epi-read0-done"}
FWD_NAMES = {0: "P.q_empty", 1: "P.kv_empty", 2: "P.item_empty", 8: "M.q_full", 9: "M.load_item", 10: "M.kv_full",
             11: "M.o_empty", 12: "M.p_full", 16: "X.s_full", 18: "X.o_done"}
COL = {"P": 0, "S": 1, "M": 1, "X": 2, "G": 3, "D": 4}


def main():
    path = sys.argv[1]
    first = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    count = int(sys.argv[3]) if len(sys.argv) > 3 else 2
    global NAMES
    ev = sorted(tuple(map(int, ln.split())) for ln in open(path) if ln.strip())
    fwd = "fwd" in path
    if fwd:
        NAMES = FWD_NAMES
    starts = [t for t, c in ev if c == (1000 if fwd else 50)]
    lo = starts[min(first, len(starts) - 1)]
    hi = starts[min(first + count, len(starts) - 1)] if first + count < len(starts) else ev[-1][0]
    open_w = {}
    print(f"items {first}..{first + count - 1}: {hi - lo} cycles ({(hi - lo) / 1.9e3:.2f} us @1.9GHz)")
    for t, c in ev:
        if c < 1000 and (fwd or c not in (50, 56, 57, 58, 82, 83, 84, 85, 66, 74, 75)):
            open_w[c] = t
            continue
        if not (lo <= t <= hi):
            continue
        base = c - 1000 if c >= 1000 else c
        name = NAMES.get(base, str(base))
        extra = f" +{t - open_w.get(base, t)}" if c >= 1000 else ""
        print(f"{t - lo:9d} " + " " * (22 * COL.get(name[0], 5)) + name + extra)


if __name__ == "__main__":
    main()
