"""Count the FP64 operations of the reference's generated residual kernels
under per-statement common-subexpression elimination (build container only:
imports the read-only reference).

The reference renders one numba kernel per plan (codegen.py:156-179): one
assignment statement per local and per residual.  LLVM (fastmath=False) may
merge identical loads and identical floating-point operations only where no
store intervenes; every residual statement ends with a store to an output
array that may alias the inputs, so merging happens *within* a statement,
not across them.  This script hash-conses each statement's expression tree
(identical operator + identical operands = one operation) and counts the
distinct +,-,*,/ nodes: the model's executed FP count per point.
2.1 measured (disassembly of a serial recompile): BL 189, RA 1065, SN 750,
SS 585 executed FP ops per point.

    PYTHONPATH=/root/reference/pkg/src FDNS_CACHE_DIR=/tmp/fdns_cache \\
        python tools/ref_cse_count.py
"""
import ast
import json

from fdns import codegen, plan, terms


def count_statement(expr, seen=None):
    seen = {} if seen is None else seen
    ops = {"n": 0}

    def key(node):
        if isinstance(node, ast.BinOp):
            k = ("bin", type(node.op).__name__, key(node.left), key(node.right))
            if k not in seen:
                seen[k] = True
                ops["n"] += 1
            return k
        if isinstance(node, ast.UnaryOp):
            return ("un", type(node.op).__name__, key(node.operand))
        return ("leaf", ast.dump(node))

    key(expr)
    return ops["n"], len(seen)


def count_plan(name):
    spec = terms.build_residual_spec()
    p = plan.build_plan(name)
    storage = plan.plan_storage(p, spec) if "spec" in plan.plan_storage.__code__.co_varnames \
        else plan.plan_storage(p)
    src = codegen.kernel_source(spec, storage)
    tree = ast.parse(src)
    total_cse, total_raw, total_region = 0, 0, 0
    per = []
    region = {}   # hash-consed ops since the last array store
    for node in ast.walk(tree):
        if isinstance(node, ast.Assign):
            raw = sum(isinstance(x, ast.BinOp) for x in ast.walk(node.value))
            if raw == 0:
                continue
            n_cse, _ = count_statement(node.value)
            n_reg, _ = count_statement(node.value, region)
            tgt = ast.unparse(node.targets[0])
            per.append((tgt, raw, n_cse))
            total_cse += n_cse
            total_raw += raw
            total_region += n_reg
            if isinstance(node.targets[0], ast.Subscript):
                region = {}   # a store into an output array ends the region
    return total_raw, total_cse, total_region, per


def main():
    out = {}
    for name in plan.PLAN_NAMES:
        raw, cse, reg, per = count_plan(name)
        out[name] = {"source_flops": raw, "per_statement_cse_flops": cse,
                     "store_region_cse_flops": reg,
                     "statements": [(t, r, c) for t, r, c in per
                                    if t.split("[")[0].startswith("d_")]}
        print(f"{name}: source {raw}, per-statement CSE {cse}, "
              f"store-region CSE {reg}")
    print(json.dumps(out))


if __name__ == "__main__":
    main()
