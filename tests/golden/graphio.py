"""Tiny JSON+npz serialisation of IR graphs for the golden fixtures.

Graph structure goes to JSON; every numpy array attribute is stored in the
companion npz under ``"<node id>/<attr path>"``.  Works for both this repo's
Graph and the reference's neoplan.Graph (same field names)."""

from __future__ import annotations

import json

import numpy as np


def _encode(value, key, arrays):
    if isinstance(value, np.ndarray):
        arrays[key] = value
        return {"__array__": key}
    if isinstance(value, dict):
        return {k: _encode(v, f"{key}.{k}", arrays) for k, v in value.items()}
    if isinstance(value, (list, tuple)):
        return {"__seq__": [_encode(v, f"{key}.{i}", arrays) for i, v in enumerate(value)],
                "tuple": isinstance(value, tuple)}
    if isinstance(value, (np.integer,)):
        return int(value)
    if isinstance(value, (np.floating,)):
        return float(value)
    return value


def _decode(value, arrays):
    if isinstance(value, dict):
        if "__array__" in value:
            return np.asarray(arrays[value["__array__"]])
        if "__seq__" in value:
            seq = [_decode(v, arrays) for v in value["__seq__"]]
            return tuple(seq) if value.get("tuple") else seq
        return {k: _decode(v, arrays) for k, v in value.items()}
    return value


def dump_graph(g, prefix: str, arrays: dict) -> dict:
    nodes = []
    for nid in sorted(g.nodes):
        n = g.nodes[nid]
        nodes.append({"id": nid, "kind": getattr(n.kind, "value", n.kind),
                      "inputs": [list(e) for e in n.inputs],
                      "attrs": _encode(dict(n.attrs), f"{prefix}/{nid}", arrays)})
    return {"name": g.name, "outputs": list(g.outputs), "nodes": nodes}


def load_graph(doc: dict, arrays, graph_cls, node_cls, kind_cls):
    g = graph_cls(doc["name"])
    for nd in doc["nodes"]:
        attrs = _decode(nd["attrs"], arrays)
        g.add_node(node_cls(nd["id"], kind_cls(nd["kind"]), attrs,
                            [tuple(e) for e in nd["inputs"]]))
    g.outputs = list(doc["outputs"])
    return g


def save(path_json: str, path_npz: str, doc: dict, arrays: dict) -> None:
    with open(path_json, "w") as fh:
        json.dump(doc, fh, indent=1, sort_keys=True)
    np.savez_compressed(path_npz, **arrays)
