"""Generate golden fixtures by running the REAL reference package.

Run in the build container (where /root/reference exists):
    python tests/golden/make_golden.py
It imports ``adacluster`` from /root/reference/pkg/src (read-only, never
copied), runs it single-threaded (threadpool_limits(1), the reference's own
determinism setting) on small seeded inputs, and stores inputs + outputs in
``tests/golden/*.npz``.  The CPU suite pins the oracle to these files
(tests/test_oracle_golden.py); the GPU suite compares the CUDA path to the
oracle at every size.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent


def main():
    sys.path.insert(0, str(REF))
    import adacluster as R
    import adacluster.quest as RQ
    from adacluster.harness.config import LayerSpec
    from adacluster.harness.synthetic import gen_synthetic
    from threadpoolctl import threadpool_limits

    meta = {"numpy": np.__version__}
    with threadpool_limits(1):
        # ---- kmeans (clustering.py:155) ----
        km = {}
        cases = [(6, 3, 6, 1), (12, 2, 2, 2), (20, 4, 1, 0), (40, 2, 15, 0), (60, 6, 5, 3),
                 (200, 8, 10, 4), (300, 64, 8, 2), (500, 32, 16, 1), (1000, 64, 20, 3),
                 (700, 17, 9, 11), (1500, 128, 24, 5)]
        for i, (n, d, k, seed) in enumerate(cases):
            rng = np.random.default_rng(seed + 100)
            x = (rng.normal(size=(n, d)) * 3).astype(np.float32)
            m = R.kmeans(x, k, seed=seed)
            km[f"c{i}_x"] = x
            km[f"c{i}_meta"] = np.array([n, d, k, seed, m.n_iter], np.int64)
            km[f"c{i}_centers"] = m.centers
            km[f"c{i}_labels"] = m.assignments
            km[f"c{i}_counts"] = m.counts
            km[f"c{i}_inertia"] = np.array(m.inertia_history, np.float64)
        np.savez_compressed(OUT / "kmeans.npz", **km)

        # ---- queries / tau / multi-stage (clustering.py:182-320) ----
        ms = {}
        spec7 = LayerSpec(kind="compact", gaussian_components=32, component_sigma=1.0,
                          component_separation=80.0, scale_spread=0.3)
        q, k, v = gen_synthetic(spec7, 2048, 64, 1, 1, 0)[0][0]
        qm, reps = R.cluster_queries(q, 65, 0)
        s0 = R.kmeans(k, 100, 0)
        tau = R.compute_tau(k, s0)
        mk = R.multi_stage_cluster_keys(k, tau, stage0=s0)
        ms.update(crit7_q=q, crit7_k=k, crit7_qlabels=qm.assignments, crit7_qcenters=qm.centers,
                  crit7_reps=reps, crit7_qiters=np.array([qm.n_iter]),
                  crit7_s0labels=s0.assignments, crit7_s0centers=s0.centers,
                  crit7_tau=np.array([tau]), crit7_mlabels=mk.assignments,
                  crit7_mcenters=mk.centers, crit7_mse=np.array(mk.stage_mse),
                  crit7_mmeta=np.array([mk.stage_count, mk.n_iter, int(mk.flag_full)]))
        for name, (kind, L, D, m0, nmax) in {
                "mixed": ("mixed", 1024, 16, 16, 200),
                "disp": ("dispersed", 512, 8, 16, 64),
                "comp": ("compact", 512, 8, 16, 1000)}.items():
            spec = LayerSpec(kind=kind, gaussian_components=8, component_sigma=0.5,
                             component_separation=20.0)
            _, kk, _ = gen_synthetic(spec, L, D, 1, 1, 3)[0][0]
            s0 = R.kmeans(kk, m0, 1)
            tau = R.compute_tau(kk, s0)
            mk = R.multi_stage_cluster_keys(kk, tau, n_max=nmax, m0=m0, seed=1, stage0=s0)
            ms[f"{name}_k"] = kk
            ms[f"{name}_args"] = np.array([m0, nmax], np.int64)
            ms[f"{name}_tau"] = np.array([tau])
            ms[f"{name}_labels"] = mk.assignments
            ms[f"{name}_centers"] = mk.centers
            ms[f"{name}_mse"] = np.array(mk.stage_mse)
            ms[f"{name}_meta"] = np.array([mk.stage_count, mk.n_iter, int(mk.flag_full)])
        np.savez_compressed(OUT / "multistage.npz", **ms)

        # ---- selection (quest.py) ----
        sel = {}
        for i, (gq, c, d) in enumerate([(2, 3, 4), (8, 16, 32), (5, 7, 11), (65, 100, 64),
                                        (30, 30, 64), (65, 17, 64)]):
            rng = np.random.default_rng(gq * 100 + c)
            x = rng.normal(size=(c * 4, d)).astype(np.float32)
            m = R.kmeans(x, c, seed=0)
            env = R.build_envelopes(x, m)
            qr = rng.normal(size=(gq, d)).astype(np.float32)
            sc = R.tensor_quest(qr, env)
            s = R.select_topk_clusters(sc, min(3, c), m.counts)
            sel[f"c{i}_x"] = x
            sel[f"c{i}_labels"] = m.assignments
            sel[f"c{i}_counts"] = m.counts
            sel[f"c{i}_reps"] = qr
            sel[f"c{i}_emax"] = env.max_vec
            sel[f"c{i}_emin"] = env.min_vec
            sel[f"c{i}_quest"] = sc
            sel[f"c{i}_mean"] = R.mean_center_scores(qr, m.centers)
            sel[f"c{i}_clamped"] = RQ.tensor_quest_clamped_centers(qr, m.centers)
            sel[f"c{i}_selected"] = s.selected
            sel[f"c{i}_density"] = np.array([s.density])
        np.savez_compressed(OUT / "selection.npz", **sel)

        # ---- pipeline (pipeline.py); inputs are regenerated by the tests with the
        # generator restatement, which synthetic.npz pins bit-for-bit ----
        pl = {}
        p = R.PipelineParams(q_clusters=65, topk=25, full_layer_quota=0.0)
        q, k, v = gen_synthetic(spec7, 4096, 64, 1, 1, 0)[0][0]
        out, hs = R.adacluster_attention(q, k, v, R.LayerPolicy(topk=25), R.StepState(), 0, p)
        pl.update(head_out=out, head_sel=hs.selection.selected,
                  head_density=np.array([hs.density]),
                  head_iters=np.array([hs.key_iters, hs.query_iters, hs.num_key_clusters]))
        spec = LayerSpec(kind="compact", gaussian_components=8, component_sigma=0.3,
                         component_separation=15.0, drift_sigma=0.02)
        layers = [gen_synthetic(spec, 256, 8, 2, 3, 2 + l) for l in range(2)]
        inputs = [[layers[l][t] for l in range(2)] for t in range(3)]
        pp = R.PipelineParams(q_clusters=8, topk=3, m0=16, n_max=1000, full_layer_quota=0.15)
        res = R.run_denoise_steps(inputs, pp, seed=1)
        for t in range(3):
            for l in range(2):
                for h in range(2):
                    pl[f"ds_{t}{l}{h}_out"] = res.outputs[t][l][h]
                    hs = res.stats[t][l][h]
                    pl[f"ds_{t}{l}{h}_iters"] = np.array([hs.key_iters, hs.query_iters])
                    if hs.selection is not None:
                        pl[f"ds_{t}{l}{h}_sel"] = hs.selection.selected
        pl["ds_modes"] = np.array([1 if pol.mode == "full" else 0 for pol in res.policies])
        pl["ds_mse"] = np.array(res.mse_layer)
        np.savez_compressed(OUT / "pipeline.npz", **pl)

        # ---- synthetic generator checksums ----
        syn = {}
        for kind in ("compact", "dispersed", "mixed"):
            st = gen_synthetic(LayerSpec(kind=kind, drift_sigma=0.02), 300, 16, 2, 3, 5)
            syn[kind] = np.stack([np.stack(st[t][h]) for t in range(3) for h in range(2)])
        np.savez_compressed(OUT / "synthetic.npz", **syn)
    (OUT / "meta.json").write_text(json.dumps(meta, indent=1) + "\n")
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()
