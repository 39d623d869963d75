"""Per-statement wall time of one function (a poor man's line profiler for
host-path work): re-executes the function's source with a timestamp after
every top-level statement of its body, in the function's own module globals.

    from tools.linetime import timed_copy
    f, report = timed_copy(module_or_class, "name")
    ... call f(...) many times ...
    report(calls)
"""
import inspect
import textwrap
import time


def timed_copy(owner, name, module=None):
    fn = getattr(owner, name)
    src = textwrap.dedent(inspect.getsource(fn))
    lines = src.split("\n")
    hdr = next(i for i, l in enumerate(lines) if l.startswith("def "))
    # end of the signature: first line after hdr ending with ':'
    sig_end = next(i for i in range(hdr, len(lines)) if lines[i].rstrip().endswith(":"))
    out = lines[: sig_end + 1]
    out.append("    _T_.append((-1, _pc_()))")
    in_doc = False
    for i in range(sig_end + 1, len(lines)):
        l = lines[i]
        s = l.strip()
        top = l.startswith("    ") and not l.startswith("     ") and s
        if top and s.startswith(('"""', "'''")):
            in_doc = not (s.count('"""') == 2 or s.count("'''") == 2) if not in_doc else False
        elif in_doc and ('"""' in s or "'''" in s):
            in_doc = False
        elif top and not in_doc and not s.startswith(("#", ")", "]", "}", "else", "elif", "except", "finally",
                                                       "@", "return")):
            out.append(f"    _T_.append(({i}, _pc_()))")
        if top and s.startswith("return"):
            out.append(f"    _T_.append(({i}, _pc_()))")
        out.append(l)
    mod = module or inspect.getmodule(fn)
    ns = dict(mod.__dict__)
    T = []
    ns["_T_"], ns["_pc_"] = T, time.perf_counter
    exec("\n".join(out), ns)
    new = ns[fn.__name__]
    acc = {}

    def wrapped(*a, **k):
        T.clear()
        try:
            return new(*a, **k)
        finally:
            T.append((len(lines), time.perf_counter()))
            for (x, tx), (_, ty) in zip(T, T[1:]):
                acc[x] = acc.get(x, 0.0) + (ty - tx)

    def report(calls, top=15):
        tot = sum(acc.values())
        print(f"{name}: {1e3 * tot / calls:.3f} ms per call")
        for x, v in sorted(acc.items(), key=lambda kv: -kv[1])[:top]:
            txt = lines[x].strip()[:90] if x >= 0 else "(entry)"
            print(f"  {1e3 * v / calls:8.3f} ms  {txt}")
        acc.clear()

    return wrapped, report
