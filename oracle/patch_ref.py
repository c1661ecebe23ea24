"""Copy the reference `partir` sources into oracle/_ref/src and apply the
three correctness patches SURVEY.md Appendix A describes.

TEST INFRASTRUCTURE ONLY: the output is the parity oracle; nothing under
oracle/ is linked into the product library.

The reference is never edited in place (it is read-only); the copy lives in
oracle/_ref/ which is git-ignored and travels to the GPU box as a build
artefact.  Each patch is an exact, anchored string replacement that must match
exactly once, so a changed reference fails loudly here instead of silently
producing a different oracle.

  A  propagate.cc:82-101  keep the PropagationRule alive while `plan.driving_class`
                          points into it (use-after-free at propagate.cc:196).
  B  spmd.cc:270,315      instantiate the registry on per-iteration LOCAL shapes
                          and lift sharded result dims back to GLOBAL.
  C  propagate.cc:179,365 shrink relocated `slice` limits on the tiled
                          pass-through dim (forward and backward).
"""
import os
import shutil
import sys

REF = os.environ.get("PARTIR_REF", "/root/reference/proj")
HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "_ref", "src")

PATCHES = {
    "src/propagate.cc": [
        # A: include for shared_ptr
        ("#include <utility>\n",
         "#include <utility>\n#include <memory>\n"),
        # A: own the rule inside the plan
        ("  struct PullPlan {\n    bool ok = false;\n",
         "  struct PullPlan {\n    std::shared_ptr<PropagationRule> rule_holder;\n    bool ok = false;\n"),
        ("    PropagationRule rule = rule_for(X, operand_types(X));\n    // Any blocked use",
         "    plan.rule_holder = std::make_shared<PropagationRule>(rule_for(X, operand_types(X)));\n"
         "    PropagationRule& rule = *plan.rule_holder;\n    // Any blocked use"),
        # C (forward): end of build_sliced_consumer
        ("      consumer.operands[m.operand] = it->second;\n    }\n  }\n",
         "      consumer.operands[m.operand] = it->second;\n    }\n"
         "    if (X.kind == OpKind::kSlice && C.role == DimRole::kPassThrough)\n"
         "      for (const DimClassMember& m : C.members)\n"
         "        consumer.limit[m.dim] = consumer.start[m.dim] +\n"
         "            (consumer.limit[m.dim] - consumer.start[m.dim]) / axis_size;\n"
         "  }\n"),
        # C (backward)
        ("          replacement.push_back(std::move(local));\n",
         "          if (P.kind == OpKind::kSlice)\n"
         "            for (const DimClassMember& m : C->members)\n"
         "              local.limit[m.dim] = local.start[m.dim] +\n"
         "                  (local.limit[m.dim] - local.start[m.dim]) / axis_size;\n"
         "          replacement.push_back(std::move(local));\n"),
    ],
    "src/spmd.cc": [
        # B: per-iteration (local) shapes for the registry
        ("    for (Lowered* v : ins) per_iter_types.push_back(v->global);\n",
         "    for (Lowered* v : ins) per_iter_types.push_back(TensorType{v->local(p.mesh)});\n"),
        # B: lift sharded dims back to global
        ("    Operation local = op;\n    for (size_t i = 0; i < ins.size(); ++i) local.operands[i]",
         "    for (size_t d = 0; d < r.spec.dim_axes.size(); ++d)\n"
         "      if (!r.spec.dim_axes[d].empty())\n"
         "        r.global.shape[d] *= p.mesh.axis_size(r.spec.dim_axes[d]);\n"
         "    Operation local = op;\n    for (size_t i = 0; i < ins.size(); ++i) local.operands[i]"),
    ],
}


def main() -> int:
    if not os.path.isdir(REF):
        print(f"patch_ref: reference not found at {REF}", file=sys.stderr)
        return 2
    if os.path.isdir(OUT):
        shutil.rmtree(OUT)
    shutil.copytree(os.path.join(REF, "include"), os.path.join(OUT, "include"))
    shutil.copytree(os.path.join(REF, "src"), os.path.join(OUT, "src"))
    for rel, edits in PATCHES.items():
        path = os.path.join(OUT, rel)
        with open(path) as f:
            text = f.read()
        for old, new in edits:
            n = text.count(old)
            if n != 1:
                print(f"patch_ref: anchor matched {n} times in {rel}:\n{old}", file=sys.stderr)
                return 3
            text = text.replace(old, new)
        with open(path, "w") as f:
            f.write(text)
    print(f"patch_ref: patched copy at {OUT}")
    return 0


if __name__ == "__main__":
    sys.exit(main())
