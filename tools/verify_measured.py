"""The paper's schedule inequalities (Eq. 3-11) checked against collective times MEASURED on B200.

    python tools/verify_measured.py profiles/nvlink_profile_p4.csv --layout 2,2,2 > profiles/verify_p4.txt

The reference checks the five closed-form claims against its simulated two-channel link model
(moesched timing.py:356-416, `moesched verify`).  Here every term comes from the alpha-beta
profile fitted to NCCL-over-NVLink measurements on the box (paper_2407_00599_b200/calibrate.py),
so the check says which of the paper's dominance claims survive on one NVSwitch box.
"""

from __future__ import annotations

import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2407_00599_b200.selector import (KEY_A2A_EP, KEY_A2A_EPESP, KEY_AG_ESP, KEY_AG_MP, KEY_AR_ESP,  # noqa: E402
                                            KEY_OVERLAP, KEY_RS_ESP, load_profile)


def main(argv=None) -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("profile")
    ap.add_argument("--layout", default="2,2,2", help="MP,EP,ESP")
    args = ap.parse_args(argv)
    mp, ep, esp = (int(v) for v in args.layout.split(","))
    prof = load_profile(args.profile)
    g = prof.get
    rows = []
    for e in range(14, 27, 2):
        x = float(2 ** e)
        a2a_fused, ag_esp, rs_esp, a2a_ep = g(KEY_A2A_EPESP)(x), g(KEY_AG_ESP)(x), g(KEY_RS_ESP)(x), g(KEY_A2A_EP)(x)
        rows.append(("fused_vs_gather_then_exchange", x, a2a_fused, ag_esp + a2a_ep, "<="))
        rows.append(("single_node_exchange_equality", x, a2a_fused, a2a_ep, "=="))
        rows.append(("fused_vs_scatter_then_exchange", x, a2a_fused, rs_esp + a2a_ep, "<="))
        disp = x * esp
        t_base = g(KEY_AG_ESP)(disp) + g(KEY_AR_ESP)(disp) + 2 * g(KEY_A2A_EP)(disp)
        t_fused = 2 * g(KEY_A2A_EPESP)(disp)
        rows.append(("fused_gain_covers_input_gather", x, g(KEY_AG_ESP)(disp), t_base - t_fused, "<="))
        if mp >= 2:
            shard = disp / mp
            t_d2 = g(KEY_A2A_EPESP)(shard) + g(KEY_OVERLAP)(shard) + g(KEY_AG_MP)(disp / esp / mp * mp)
            rows.append(("overlap_never_worse_than_baseline", x, t_d2, t_base, "<="))
    print(f"profile {args.profile}, layout MP={mp} EP={ep} ESP={esp} (single NVSwitch box)")
    print(f"{'claim':36s} {'elements':>10s} {'lhs us':>10s} {'rhs us':>10s}  holds")
    summary = {}
    for name, x, lhs, rhs, op in rows:
        ok = (abs(lhs - rhs) <= 0.05 * max(lhs, rhs)) if op == "==" else lhs <= rhs * 1.0000001
        summary.setdefault(name, [0, 0])
        summary[name][0] += ok
        summary[name][1] += 1
        print(f"{name:36s} {x:10.0f} {lhs * 1e6:10.1f} {rhs * 1e6:10.1f}  {'yes' if ok else 'NO'}"
              f"{' (within 5%)' if op == '==' else ''}")
    print()
    for name, (ok, n) in summary.items():
        print(f"{name:36s} holds at {ok}/{n} sizes")
    return 0


if __name__ == "__main__":
    sys.exit(main())
