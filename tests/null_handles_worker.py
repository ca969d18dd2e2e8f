"""Calls every handle-taking entry point of include/ginsim_cuda.h with null
handles (and a one-element handle list holding null) and prints the ones that
did not answer GINSIM_E_USAGE (destroy functions: GINSIM_OK).  Run in a
subprocess by tests/test_descriptor_abi.py so a crash fails one test instead
of the whole session.  CPU only: every call must fail before touching the
device."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_15076_b200 as G  # noqa: E402

# entry points without a comm / moe / plugin handle first
SKIP = ("wire_", "inproc_", "socket_", "descriptor_", "config_", "last_error", "abi_version", "reserve_loopback",
        "occupy", "comm_create")


def main():
    L = G.lib()
    bad, n = [], 0
    for name in G.exported_symbols():
        if any(s in name for s in SKIP):
            continue
        fn = getattr(L, name)
        if not fn.argtypes:  # not bound from Python (the plugin entry points: test_descriptor_abi.py)
            continue
        args = []
        for k, t in enumerate(fn.argtypes or []):
            if t is ctypes.c_void_p or t is ctypes.c_char_p:
                args.append(None)
            elif k == 0 and t is ctypes.POINTER(ctypes.c_void_p):
                args.append((ctypes.c_void_p * 8)())  # a handle list of nulls
            elif hasattr(t, "_type_") and not isinstance(t._type_, str):
                args.append(None)  # out-pointers / structs
            else:
                args.append(1)  # counts, ids, sizes: 1 gets past the shape checks
        rc = fn(*args)
        n += 1
        want = 0 if name.endswith("_destroy") else 23
        if rc != want:
            bad.append(f"{name}: {rc}")
    print(f"checked {n}")
    print("BAD " + "; ".join(bad) if bad else "all null handles rejected")


if __name__ == "__main__":
    main()
