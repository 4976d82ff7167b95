"""Tool-side convenience: map MOE_B200_<OPTION> environment variables onto the
library's debug options (moe_debug_set_option).  The product library itself
never reads the environment; only these measurement tools do, through here."""
import os

NAMES = ["stack", "stack_kernel", "rw", "prefill", "prefill_splits", "stack_grid", "virtual_stack",
         "noncoop", "force_ep", "no_pdl", "combine4", "pf_debug", "pf_evict", "pf_lag", "pf_late8",
         "pf_slo", "pf_persist"]


def from_env():
    import paper_2402_07033_b200 as M

    applied = {}
    for n in NAMES:
        v = os.environ.get("MOE_B200_" + n.upper())
        if v is not None and v != "":
            M.set_option(n, int(v))
            applied[n] = int(v)
    tp = os.environ.get("MOE_B200_PF_TRACE")
    if tp:
        M.set_trace_path(tp)
        applied["pf_trace"] = tp
    return applied
