"""Bridge to the unmodified reference package ``neoplan`` -- TEST / BASELINE
INFRASTRUCTURE ONLY.

The reference is pure Python + numba (no build step).  It is found either
installed under ``baseline/_ref`` (``pip install --target baseline/_ref``
of /root/reference/pkg, git-ignored; travels to the GPU box) or, in the
build container only, straight from /root/reference/pkg/src.  It is used to
generate the golden fixtures (tests/golden/make_golden.py) and as the CPU
baseline arm of bench.py; the product package never touches it.
"""

from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CANDIDATES = (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src")


def import_reference():
    """Return the ``neoplan`` module or raise ImportError."""
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/neoplan_numba_cache")
    for path in CANDIDATES:
        if os.path.isdir(os.path.join(path, "neoplan")):
            if path not in sys.path:
                sys.path.insert(0, path)
            import neoplan  # noqa: F401
            return neoplan
    raise ImportError("reference package neoplan not found (baseline/_ref missing)")


def reference_location() -> str | None:
    for path in CANDIDATES:
        if os.path.isdir(os.path.join(path, "neoplan")):
            return path
    return None


def to_reference_graph(g, neoplan):
    """Copy a graph built with this repo's IR into a ``neoplan.Graph``
    (same operator names, attributes and node ids).  Only graphs with scalar
    stride/pad are expressible in the reference."""
    ng = neoplan.Graph(g.name)
    for nid in sorted(g.nodes):
        node = g.nodes[nid]
        kind = neoplan.OpKind(node.kind.value)
        attrs = dict(node.attrs)
        for key in ("stride", "pad"):
            if isinstance(attrs.get(key), (tuple, list)):
                a, b = attrs[key]
                if a != b:
                    raise ValueError(f"node {nid}: asymmetric {key} {attrs[key]} is not "
                                     "expressible in the reference")
                attrs[key] = int(a)
        ng.add_node(neoplan.graph.Node(nid, kind, attrs, list(node.inputs)))
    ng.outputs = list(g.outputs)
    return ng


def reference_optimized(ng, neoplan):
    """The reference's optimized pipeline: simplify -> uniform assignment ->
    alter layouts -> pre-pack weights (passes.py:373, :325, :167, :258)."""
    s = neoplan.simplify(ng)
    assign = neoplan.uniform_assignment(s)
    return neoplan.pretransform_weights(neoplan.alter_and_insert_transforms(s, assign))
