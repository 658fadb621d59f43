"""Data link, mirroring peakmem.linking (pkg/src/peakmem/linking.py).

The three joins -- innermost non-wrapper layer per root operator
(linking.py:50-65), backward operators by sequence number (linking.py:68-92)
and block -> owning operator / layer with the temporary / retained split
(linking.py:95-123) -- run in `pm_link` (csrc/pipeline.cu).  This module
turns the columnar result into LayerMemoryProfile objects keyed by LayerNode.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _pipeline
from .analysis import (BlockRole, LayerNode, MemoryBlock, OperatorNode,
                       blocks_from_link)

class ProfileMap(dict):
    """dict[LayerNode, LayerMemoryProfile] (linking.py:24) that also
    remembers the roots it was linked over and whether backward operators
    are attached, so the step functions below can each re-run the device
    join on the same inputs."""

    roots: list | None = None
    backward_attached: bool = False


@dataclass(eq=False)
class LayerMemoryProfile:
    """Per-layer view (linking.py:27-43)."""

    layer: LayerNode
    forward_ops: list[OperatorNode] = field(default_factory=list)
    backward_ops: list[OperatorNode] = field(default_factory=list)
    retained_blocks: list[MemoryBlock] = field(default_factory=list)
    temporary_blocks: list[MemoryBlock] = field(default_factory=list)

    def owned_ops(self) -> list[OperatorNode]:
        return self.forward_ops + self.backward_ops

    def backward_retained_blocks(self) -> list[MemoryBlock]:
        """Retained blocks allocated during this layer's backward ops."""
        return [b for b in self.retained_blocks
                if any(op.contains_ts(b.alloc_time) for op in self.backward_ops)]


def non_wrapper_layers(tree: LayerNode) -> list[LayerNode]:
    """Leaves in pre-order walk order (linking.py:46-47)."""
    return [n for n in tree.walk() if n is not tree and not n.is_wrapper]


def profiles_from_link(leaves: list[LayerNode], roots: list[OperatorNode],
                       blocks: list[MemoryBlock], link) -> ProfileMap:
    profiles = ProfileMap((leaf, LayerMemoryProfile(leaf)) for leaf in leaves)
    for r, w in enumerate(link.root_leaf.tolist()):
        if w >= 0:
            profiles[leaves[w]].forward_ops.append(roots[r])
    off = link.bwd_off.tolist()
    bw = link.bwd_root.tolist()
    for w, leaf in enumerate(leaves):
        profiles[leaf].backward_ops = [roots[r] for r in bw[off[w]:off[w + 1]]]
    for b, (role, prof) in enumerate(zip(link.b_role.tolist(),
                                         link.b_prof.tolist())):
        if prof < 0:
            continue
        p = profiles[leaves[prof]]
        (p.temporary_blocks if role == 5 else p.retained_blocks).append(blocks[b])
    return profiles


def _join(leaves, roots, blocks=(), with_seqs=True):
    seq_off = [0]
    seqs: list[int] = []
    for op in roots:
        if with_seqs:
            seqs.extend(sorted(op.sequence_numbers))
        seq_off.append(len(seqs))
    none = _pipeline.NONE
    return _pipeline.link_roots(
        [op.start_ts for op in roots], [op.end_ts for op in roots], seq_off,
        seqs, [n.start_ts for n in leaves], [n.end_ts for n in leaves],
        [b.alloc_time for b in blocks],
        [none if b.free_time is None else b.free_time for b in blocks])


def link_layers_to_ops(tree: LayerNode, roots: list[OperatorNode]) -> ProfileMap:
    """Each root operator to the innermost non-wrapper layer containing it
    (linking.py:50-65), on the device (sorted-leaf probe in pm_link_roots)."""
    leaves = non_wrapper_layers(tree)
    profiles = ProfileMap((leaf, LayerMemoryProfile(leaf)) for leaf in leaves)
    profiles.roots = list(roots)
    if leaves and roots:
        lk = _join(leaves, roots, with_seqs=False)
        for r, w in enumerate(lk.root_leaf.tolist()):
            if w >= 0:
                profiles[leaves[w]].forward_ops.append(roots[r])
    return profiles


def attach_backward_ops(profiles: ProfileMap,
                        all_ops: list[OperatorNode]) -> ProfileMap:
    """Per layer, every other operator carrying one of its forward
    sequence numbers, ordered by start (linking.py:68-92), via the device
    sequence-number join.  The forward ownership is the device's own
    link_layers_to_ops over `all_ops` (the reference passes the same list
    to both steps, linking.py:129-130)."""
    leaves = list(profiles)
    if leaves and all_ops:
        lk = _join(leaves, all_ops)
        off = lk.bwd_off.tolist()
        bw = lk.bwd_root.tolist()
        for w, leaf in enumerate(leaves):
            profiles[leaf].backward_ops = [all_ops[r] for r in bw[off[w]:off[w + 1]]]
    else:
        for p in profiles.values():
            p.backward_ops = []
    if isinstance(profiles, ProfileMap):
        profiles.roots = list(all_ops)
        profiles.backward_attached = True
    return profiles


def attach_blocks(profiles: ProfileMap,
                  blocks: list[MemoryBlock]) -> ProfileMap:
    """Each block to the layer owning the operator it was born in, as an
    intra-operator temporary or retained (linking.py:95-123), via the
    device owner join; roles are set in place like the reference."""
    leaves = list(profiles)
    roots = getattr(profiles, "roots", None)
    with_bwd = getattr(profiles, "backward_attached", None)
    if roots is None:  # a plain dict: its owned operators are the roots
        seen: set[int] = set()
        roots = []
        for p in profiles.values():
            for op in p.owned_ops():
                if id(op) not in seen:
                    seen.add(id(op))
                    roots.append(op)
        with_bwd = any(p.backward_ops for p in profiles.values())
    if not (leaves and roots and blocks):
        return profiles
    lk = _join(leaves, roots, blocks, with_seqs=bool(with_bwd))
    for b, role, prof in zip(blocks, lk.b_role.tolist(), lk.b_prof.tolist()):
        if prof < 0:
            continue
        p = profiles[leaves[prof]]
        if role == 5:
            b.role = BlockRole.TEMPORARY
            p.temporary_blocks.append(b)
        else:
            b.role = BlockRole.RETAINED
            p.retained_blocks.append(b)
    return profiles


def link(tree: LayerNode, roots: list[OperatorNode],
         blocks: list[MemoryBlock]) -> ProfileMap:
    """Run the three linking steps (linking.py:126-132) on the GPU over the
    given roots and blocks; sets block roles in place, like the reference."""
    leaves = non_wrapper_layers(tree)
    profiles = ProfileMap((leaf, LayerMemoryProfile(leaf)) for leaf in leaves)
    profiles.roots = list(roots)
    profiles.backward_attached = True
    if not (leaves and roots):
        return profiles
    lk = _join(leaves, roots, blocks)
    for r, w in enumerate(lk.root_leaf.tolist()):
        if w >= 0:
            profiles[leaves[w]].forward_ops.append(roots[r])
    off = lk.bwd_off.tolist()
    bw = lk.bwd_root.tolist()
    for w, leaf in enumerate(leaves):
        profiles[leaf].backward_ops = [roots[r] for r in bw[off[w]:off[w + 1]]]
    for b, role, prof in zip(blocks, lk.b_role.tolist(), lk.b_prof.tolist()):
        if prof < 0:
            continue
        p = profiles[leaves[prof]]
        if role == 5:
            b.role = BlockRole.TEMPORARY
            p.temporary_blocks.append(b)
        else:  # retained (3 = retained and backward: a gradient candidate)
            b.role = BlockRole.RETAINED
            p.retained_blocks.append(b)
    return profiles


__all__ = ["LayerMemoryProfile", "ProfileMap", "attach_backward_ops",
           "attach_blocks", "link", "link_layers_to_ops", "non_wrapper_layers",
           "profiles_from_link", "blocks_from_link"]
