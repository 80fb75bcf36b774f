"""Topologies, communication sketches and the alpha-beta cost model (§3-§4).

* alpha-beta model: a chunk of s MB over link l costs alpha_l + beta_l * s;
  k chunks sent together cost alpha + k*beta*s.
* Table 1 gives V100-era constants; the B200 NVLink beta below is the
  nominal 900 GB/s per direction (1 MiB / 900 GB/s = 1.165 us), alpha stays the table's
  0.7 us until the NVLink 5 profiler measures it.
* A communication sketch (Listing 1 at 1289–1315) restricts the physical
  topology to a logical one: switch-hyperedge policy (uc-max / uc-min),
  inter-node connections, beta_split, chunk-to-relay map, rotational symmetry offsets,
  input_chunkup and input_size.
"""
from __future__ import annotations

import json
import re
from dataclasses import dataclass, field

NVLINK_ALPHA_US = 0.7            # Table 1
NVLINK5_BETA_US_PER_MB = (1 << 20) / 900e9 * 1e6   # 1.165 us/MB at 900 GB/s
IB_ALPHA_US, IB_BETA_US_PER_MB = 1.7, 106.0        # Table 1
# Measured on this pool's B200s the paper's way (k chunks one after another
# vs all at once on one link, least squares; tools/ab_profile.py through this executor,
# generator/profiler.py, profiles/r02_alphabeta.json): zero-copy kernel alpha 5.35 us, beta
# 1.43 us/MB (733 GB/s per connection, both directions busy), plus ~9.4 us per call; LL kernel
# (<= 2 MiB) alpha 2.58 us, beta 3.65 us/MB. The connection-count sweep (PAPER.md:405-418,
# tools/nvlink_probe.cu, profiles/r02_nvlink_probe.jsonl) at 1 GiB per GPU: 695 / 694 / 623
# GB/s accumulated egress over 1 / 2 / 3 concurrent connections (4 GPUs) — the paper's
# multi-connection effect on NVLink 5.
B200_NVLINK_ALPHA_US = 5.35
B200_NVLINK_BETA_US_PER_MB = 1.43
B200_LL_ALPHA_US, B200_LL_BETA_US_PER_MB = 2.58, 3.65


@dataclass(frozen=True)
class Link:
    alpha: float      # us
    beta: float       # us per MB (MB = 2^20 bytes)
    kind: str         # "nvlink" | "ib"

    def cost(self, mb: float, k: int = 1) -> float:
        """alpha-beta time of k chunks of `mb` MB sent together."""
        return self.alpha + k * self.beta * mb


@dataclass
class Topology:
    name: str
    n: int
    node_of: list
    links: dict = field(default_factory=dict)      # (u, v) -> Link
    switches: list = field(default_factory=list)   # rank lists sharing a switch (hyperedges)

    def per_node(self):
        return self.n // (max(self.node_of) + 1)


def nvswitch(n: int, alpha=NVLINK_ALPHA_US, beta=NVLINK5_BETA_US_PER_MB) -> Topology:
    """One B200 NVSwitch domain: every GPU reaches every other at full bandwidth. Defaults are
    the paper's alpha with the nominal NVLink 5 beta; nvswitch_measured() uses the profile."""
    t = Topology(f"nvswitch{n}", n, [0] * n)
    for u in range(n):
        for v in range(n):
            if u != v:
                t.links[(u, v)] = Link(alpha, beta, "nvlink")
    t.switches.append(list(range(n)))
    return t


def nvswitch_measured(n: int) -> Topology:
    """nvswitch() with the alpha-beta values profiled on B200 (B200_NVLINK_*)."""
    return nvswitch(n, B200_NVLINK_ALPHA_US, B200_NVLINK_BETA_US_PER_MB)


def multinode(nodes: int, per_node: int, intra=(NVLINK_ALPHA_US, NVLINK5_BETA_US_PER_MB),
              inter=(IB_ALPHA_US, IB_BETA_US_PER_MB)) -> Topology:
    """`nodes` NVSwitch nodes; every GPU may reach every remote GPU over an IB switch. On one
    B200 box this is the emulated 2x4 configuration C5 (topological only)."""
    n = nodes * per_node
    t = Topology(f"{nodes}x{per_node}", n, [r // per_node for r in range(n)])
    for u in range(n):
        for v in range(n):
            if u == v:
                continue
            same = t.node_of[u] == t.node_of[v]
            a, b = intra if same else inter
            t.links[(u, v)] = Link(a, b, "nvlink" if same else "ib")
    for nd in range(nodes):
        t.switches.append(list(range(nd * per_node, (nd + 1) * per_node)))
    return t


# ------------------------------------------------------------------------------ sketch

@dataclass
class Sketch:
    policy: str = "uc-max"                 # switch_hyperedge_strategy
    internode_conn: dict | None = None     # local i -> [local j, ...] on another node
    beta_split: dict = field(default_factory=dict)   # local i -> divisor of inter-node bw
    chunk_to_relay: tuple | None = None    # (r1, r2): relay = (rp // r1) * r1 + r2
    symmetry_offsets: list = field(default_factory=list)   # [(o, g), ...]
    input_chunkup: int = 1
    input_size: int = 1 << 20              # bytes


def _size(s) -> int:
    if isinstance(s, (int, float)):
        return int(s)
    m = re.fullmatch(r"\s*([0-9.]+)\s*([KMG]?)B?\s*", str(s), re.I)
    if not m:
        raise ValueError(f"bad size {s!r}")
    return int(float(m.group(1)) * {"": 1, "K": 1 << 10, "M": 1 << 20, "G": 1 << 30}[m.group(2).upper()])


def parse_sketch(text: str) -> Sketch:
    """Listing 1's JSON; // comments allowed."""
    clean = re.sub(r"//[^\n]*", "", text)
    d = json.loads(clean)
    sk = Sketch()
    intra = d.get("intranode_sketch", {})
    pol = intra.get("switch_hyperedge_strategy", ["uc-max"])
    sk.policy = pol[0] if isinstance(pol, list) else pol
    inter = d.get("internode_sketch", {})
    if "internode_conn" in inter:
        sk.internode_conn = {int(k): [int(x) for x in v] for k, v in inter["internode_conn"].items()}
    sk.beta_split = {int(k): int(v) for k, v in inter.get("beta_split", {}).items()}
    if "chunk_to_relay_map" in inter:
        r1, r2 = inter["chunk_to_relay_map"]
        sk.chunk_to_relay = (int(r1), int(r2))
    for o, g in d.get("symmetry_offsets", []):
        if not (0 < o < g):
            raise ValueError(f"symmetry offset {(o, g)}: need 0 < o < g")
        sk.symmetry_offsets.append((int(o), int(g)))
    hp = d.get("hyperparameters", {})
    sk.input_chunkup = int(hp.get("input_chunkup", 1))
    sk.input_size = _size(hp.get("input_size", 1 << 20))
    return sk


def relay_for_chunk(sk: Sketch, rp: int) -> int:
    """Listing 1: chunk c leaves its node via GPU (rp // r1) * r1 + r2."""
    r1, r2 = sk.chunk_to_relay
    return (rp // r1) * r1 + r2


def apply_sketch(topo: Topology, sk: Sketch) -> Topology:
    """Logical topology: prune inter-node links to internode_conn, scale
    inter-node beta by beta_split, and apply the switch policy: uc-max keeps every switched
    link (all pairs), uc-min keeps a ring through each switch."""
    lt = Topology(topo.name + "+sketch", topo.n, list(topo.node_of), dict(topo.links), [list(s) for s in topo.switches])
    k = topo.per_node()
    for (u, v), l in list(lt.links.items()):
        if topo.node_of[u] != topo.node_of[v]:
            if sk.internode_conn is not None and (v % k) not in sk.internode_conn.get(u % k, []):
                del lt.links[(u, v)]
                continue
            div = sk.beta_split.get(u % k, 1)
            if div != 1:
                lt.links[(u, v)] = Link(l.alpha, l.beta * div, l.kind)
    if sk.policy == "uc-min":
        for sw in topo.switches:
            ring = {(sw[i], sw[(i + 1) % len(sw)]) for i in range(len(sw))}
            for a in sw:
                for b in sw:
                    if a != b and (a, b) not in ring:
                        lt.links.pop((a, b), None)
    return lt


def rotate(rank: int, o: int, g: int) -> int:
    """Rotational symmetry: rank -> base + (rank - base + o) mod g."""
    base = (rank // g) * g
    return base + (rank - base + o) % g
