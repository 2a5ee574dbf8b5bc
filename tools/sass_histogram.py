"""Static SASS opcode histograms of the hot kernels (cuobjdump -sass of the
in-tree objects), committed under profiles/ so the tcgen05-free, TMA +
mbarrier streaming structure is checkable without re-dumping:
UBLKCP / UTMA* = bulk TMA copies, SYNCS = mbarrier ops, DFMA / DMUL = the
float64 controller.

    python tools/sass_histogram.py > profiles/r2_sass_histograms.json
"""
import collections
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OBJ = os.path.join(ROOT, "paper_2305_16510_b200", "lib", "obj")
KERNELS = {
    # (object, mangled-name regex, label)
    "stream_kernel cfg2 (velocity, FEAT 0, 20 consumer warps)":
        ("fs_step_vel.o", r"_ZN2fs13stream_kernelILi1ELb0ELi2ELi20ELi1ELi5ELi0EEEvNS_7KParamsE"),
    "stream_kernel cfg3 (position, stats + re-spawns)":
        ("fs_step_pos.o", r"_ZN2fs13stream_kernelILi3ELb0ELi2ELi20ELi1ELi5ELi3EEEvNS_7KParamsE"),
    "stream_kernel cfg4 (position, hetero, outputs)":
        ("fs_step_pos.o", r"_ZN2fs13stream_kernelILi3ELb1ELi2ELi20ELi1ELi4ELi4EEEvNS_7KParamsE"),
    "world_stream_kernel (free-space World.step, velocity)":
        ("fs_world.o", r"_ZN2fs19world_stream_kernelILi1ELi2ELi2ELi2ELi0EEEvNS_7KParamsENS_11WorldParamsE"),
    "world_stream_kernel (obstacle World.step, velocity, deferred test + resets)":
        ("fs_world.o", r"_ZN2fs19world_stream_kernelILi1ELi2ELi2ELi2ELi2EEEvNS_7KParamsENS_11WorldParamsE"),
    "world_post_kernel (deferred resets + collision tests)":
        ("fs_world.o", r"_ZN2fs17world_post_kernelENS_11WorldParamsE"),
    "render_kernel (depth camera, 1 CTA per SM)":
        ("fs_scene.o", r"_ZN2fs13render_kernelILi1EEEv8fs_scene9fs_cameraPKflPKdlliPfPi"),
}


def functions(obj):
    out = subprocess.run(["cuobjdump", "-sass", os.path.join(OBJ, obj)], capture_output=True,
                         text=True, check=True).stdout
    cur, body = None, collections.defaultdict(list)
    for line in out.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            cur = m.group(1)
            continue
        m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(.*?);", line)
        if cur and m:
            body[cur].append(m.group(1))
    return body


def histogram(insts):
    h = collections.Counter()
    for ins in insts:
        ins = re.sub(r"^@!?U?P\w+\s+", "", ins.strip())
        h[ins.split(" ")[0].split(".")[0]] += 1
    return h


def main():
    res = {}
    cache = {}
    for label, (obj, name) in KERNELS.items():
        funcs = cache.setdefault(obj, functions(obj))
        insts = funcs.get(name)
        if insts is None:
            res[label] = {"error": f"{name} not found in {obj}"}
            continue
        h = histogram(insts)
        res[label] = {"function": name, "static_instructions": len(insts),
                      "tma_bulk_copies (UBLKCP)": h.get("UBLKCP", 0),
                      "mbarrier ops (SYNCS)": h.get("SYNCS", 0),
                      "fp64 (DFMA/DMUL/DADD)": h.get("DFMA", 0) + h.get("DMUL", 0) +
                      h.get("DADD", 0),
                      "tensor-core ops (UTCMMA/HMMA)": h.get("UTCMMA", 0) + h.get("HMMA", 0),
                      "opcodes": dict(h.most_common())}
    json.dump(res, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main()
