"""Flatten / rebuild a localisation scene (map entries + query jobs) to / from npz.

Used to replay scenes generated with the reference's synth on the GPU box,
where the reference package is absent.  Rebuilt objects are the package's
own duck-compatible types (``paper_2601_04185_b200.localizer``).
"""

from __future__ import annotations

import numpy as np


def pack_scene(entries, jobs, prefix="s_"):
    out = {}
    out[prefix + "entry_ids"] = np.array([e.id for e in entries])
    for i, e in enumerate(entries):
        p = f"{prefix}e{i}_"
        out[p + "q"], out[p + "t"] = np.asarray(e.pose.q), np.asarray(e.pose.t)
        I = e.intrinsics
        out[p + "intr"] = np.array([I.fx, I.fy, I.cx, I.cy, I.width, I.height], dtype=np.float64)
        out[p + "desc"] = np.asarray(e.descriptor, dtype=np.float32)
        if e.qdepth is not None:
            out[p + "codes"] = e.qdepth.codes
            out[p + "qparams"] = np.array([e.qdepth.d_min, e.qdepth.d_max, e.qdepth.levels], dtype=np.float64)
    out[prefix + "njobs"] = np.array(len(jobs))
    for j, job in enumerate(jobs):
        p = f"{prefix}j{j}_"
        I = job.intrinsics
        out[p + "intr"] = np.array([I.fx, I.fy, I.cx, I.cy, I.width, I.height], dtype=np.float64)
        out[p + "desc"] = np.asarray(job.descriptor, dtype=np.float64)
        out[p + "kloc"] = np.array(job.k_loc)
        out[p + "qid"] = np.array(job.query_id)
        out[p + "fids"] = np.array(sorted(job.fields))
        for k, eid in enumerate(sorted(job.fields)):
            fp = job.fields[eid]
            for tag, f in (("q2db", fp.query_to_db), ("db2q", fp.db_to_query)):
                out[f"{p}f{k}_{tag}_t"] = f.targets
                out[f"{p}f{k}_{tag}_c"] = f.confidence
                out[f"{p}f{k}_{tag}_s"] = np.array([f.scale_x, f.scale_y])
    return out


def unpack_scene(z, prefix="s_"):
    from paper_2601_04185_b200.geometry import CameraIntrinsics, Pose
    from paper_2601_04185_b200.localizer import CorrespondenceField, FieldPair, QuantizedDepthMap, QueryJob

    def intr(a):
        return CameraIntrinsics(float(a[0]), float(a[1]), float(a[2]), float(a[3]), int(a[4]), int(a[5]))

    class Entry:
        pass

    entries = []
    for i, eid in enumerate(z[prefix + "entry_ids"]):
        p = f"{prefix}e{i}_"
        e = Entry()
        e.id = str(eid)
        e.pose = Pose(z[p + "q"], z[p + "t"])
        e.intrinsics = intr(z[p + "intr"])
        e.descriptor = z[p + "desc"]
        e.qdepth = None
        if p + "codes" in z:
            qp = z[p + "qparams"]
            e.qdepth = QuantizedDepthMap(z[p + "codes"], float(qp[0]), float(qp[1]), int(qp[2]), e.intrinsics)
        entries.append(e)

    class Map:
        pass

    vmap = Map()
    vmap.entries = entries
    jobs = []
    for j in range(int(z[prefix + "njobs"])):
        p = f"{prefix}j{j}_"
        fields = {}
        for k, eid in enumerate(z[p + "fids"]):
            fl = {}
            for tag in ("q2db", "db2q"):
                s = z[f"{p}f{k}_{tag}_s"]
                fl[tag] = CorrespondenceField("a", "b", z[f"{p}f{k}_{tag}_t"], z[f"{p}f{k}_{tag}_c"],
                                              float(s[0]), float(s[1]))
            fields[str(eid)] = FieldPair(query_to_db=fl["q2db"], db_to_query=fl["db2q"])
        jobs.append(QueryJob(str(z[p + "qid"]), intr(z[p + "intr"]), z[p + "desc"], fields, int(z[p + "kloc"])))
    return vmap, jobs
