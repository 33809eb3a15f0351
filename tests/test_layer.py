"""Differentiable layer (paper_2604_18780_b200/layer.py): the torch input stage and gold scores
against the numpy restatement of the reference (CPU), and the device training loss and
gradients against the reference's hand-derived formula (validation.py:388-417) on the GPU."""

from __future__ import annotations

import numpy as np
import pytest
import torch

import paper_2604_18780_b200 as scrf
from paper_2604_18780_b200 import layer
from paper_2604_18780_b200.potentials import (CenteringMode, EmissionBatch, SemiCRFParams, Segmentation,
                                             build_scores, score_segmentation)


def _instance(seed=0, B=3, T=17, K=5, C=4):
    rng = np.random.default_rng(seed)
    em = rng.uniform(-2, 2, (B, T, C))
    lengths = np.array([T, T - 4, 6][:B], dtype=np.int64)
    params = SemiCRFParams(rng.uniform(-1, 1, (C, C)), rng.uniform(-0.5, 0.5, (K, C)),
                           rng.uniform(-1, 1, C), rng.uniform(-1, 1, C))
    return em, lengths, params


def _random_tiling(rng, L, K, C):
    segs, s = [], 0
    while s < L:
        e = min(L, s + int(rng.integers(1, K + 1)))
        segs.append((s, e, int(rng.integers(0, C))))
        s = e
    return Segmentation(tuple(segs))


@pytest.mark.parametrize("mode", [CenteringMode.NONE, CenteringMode.MEAN, CenteringMode.SHARED_MAX])
def test_input_stage_matches_numpy(mode):
    em, lengths, params = _instance()
    cum = build_scores(EmissionBatch(em, lengths), params, mode)
    S = layer.build_scores_t(torch.tensor(em), torch.tensor(lengths), mode, torch.tensor(params.pi_start),
                             torch.tensor(params.pi_end))
    np.testing.assert_allclose(S.numpy(), cum.S, rtol=0, atol=1e-12)


def test_gold_scores_match_numpy():
    em, lengths, params = _instance(1)
    cum = build_scores(EmissionBatch(em, lengths), params, CenteringMode.MEAN)
    rng = np.random.default_rng(5)
    golds = [_random_tiling(rng, int(L), params.max_duration, params.num_labels) for L in lengths]
    got = layer.gold_scores_t(torch.tensor(cum.S), torch.tensor(params.transition), torch.tensor(params.duration_bias),
                              golds).numpy()
    want = [score_segmentation(cum, params, g, b) for b, g in enumerate(golds)]
    np.testing.assert_allclose(got, want, rtol=1e-13, atol=1e-12)


def test_input_stage_rejects_non_finite():
    em, lengths, _ = _instance()
    em[1, 2, 3] = np.nan
    with pytest.raises(ValueError, match="b=1, t=2, c=3"):
        layer.center_emissions_t(torch.tensor(em), torch.tensor(lengths), CenteringMode.NONE)


@pytest.mark.gpu
def test_training_loss_and_grads_match_reference_formula():
    """Autograd through the device layer == the reference's suffix-sum derivation
    (validation.py:388-417) evaluated with the parity-pinned posterior, fp64 kernels."""
    from paper_2604_18780_b200 import streaming as S

    em, lengths, params = _instance(2, B=3, T=40, K=6, C=5)
    params = SemiCRFParams(params.transition, params.duration_bias)  # no scalar boundaries
    rng = np.random.default_rng(7)
    golds = [_random_tiling(rng, int(L), params.max_duration, params.num_labels) for L in lengths]
    prev = S.get_precision()
    S.set_precision("fp64")
    try:
        nll, ge, gT, gB = layer.training_loss_and_grads_device(em, lengths, params.transition, params.duration_bias,
                                                               golds)
        cum = build_scores(EmissionBatch(em, lengths), params, CenteringMode.NONE)
        logZ, grads, _ = scrf.posterior(cum, params)
    finally:
        S.set_precision(prev)
    B, T, C = em.shape
    K = params.max_duration
    ge_model = grads.grad_S[:, :0:-1, :].cumsum(axis=1)[:, ::-1, :]
    gold = np.zeros(B)
    g_e, g_T, g_B = np.zeros((B, T, C)), np.zeros((C, C)), np.zeros((K, C))
    from paper_2604_18780_b200.potentials import segment_path_score

    for b, g in enumerate(golds):
        per_source = segment_path_score(cum, params, g, b)
        m = per_source.max()
        gold[b] = m + np.log(np.exp(per_source - m).sum())
        p_src = np.exp(per_source - gold[b])
        prev_c = None
        for s, e, c in g:
            g_e[b, s:e, c] += 1.0
            g_B[e - s - 1, c] += 1.0
            if prev_c is None:
                g_T[:, c] += p_src
            else:
                g_T[prev_c, c] += 1.0
            prev_c = c
    np.testing.assert_allclose(nll, np.mean(logZ - gold), rtol=1e-12)
    np.testing.assert_allclose(ge, (ge_model - g_e) / B, atol=1e-10)
    np.testing.assert_allclose(gT, (grads.grad_T - g_T) / B, atol=1e-10)
    np.testing.assert_allclose(gB, (grads.grad_B - g_B) / B, atol=1e-10)


def test_cli_parser_and_dense_rejection(capsys):
    from paper_2604_18780_b200 import cli

    args = cli.build_parser().parse_args(["decode", "--params", "p.json", "--emissions", "e.csv", "--backend", "dense"])
    assert args.command == "decode" and args.centering == "none"
    assert cli.main(["bench", "--backend", "dense"]) == 2
    assert '"status": "fail"' in capsys.readouterr().err


@pytest.mark.gpu
def test_cli_decode_with_marginals(tmp_path):
    """decode --marginals (cli.py:390-440): segmentations and scores equal decode(); the
    marginal document equals posterior()'s per-position marginals trimmed to each length."""
    import json

    from paper_2604_18780_b200 import cli, streaming as S
    from paper_2604_18780_b200.potentials import save_emissions_csv, save_params_json

    em, lengths, params = _instance(9, B=2, T=30, K=5, C=3)
    params = SemiCRFParams(params.transition, params.duration_bias)
    save_params_json(params, str(tmp_path / "p.json"))
    save_emissions_csv(EmissionBatch(em, lengths), str(tmp_path / "e.csv"))
    rc = cli.main(["decode", "--params", str(tmp_path / "p.json"), "--emissions", str(tmp_path / "e.csv"),
                   "--marginals", str(tmp_path / "m.json"), "--out", str(tmp_path / "d.json")])
    assert rc == 0
    doc = json.load(open(tmp_path / "d.json"))
    cum = build_scores(EmissionBatch(em, lengths), params, CenteringMode.NONE)
    segs, scores = S.decode(cum, params)
    assert doc["scores"] == [float(v) for v in scores]
    from paper_2604_18780_b200.potentials import segmentations_from_json

    assert [tuple(s) for s in segmentations_from_json(doc["segmentations"])] == [tuple(s) for s in segs]
    m = json.load(open(tmp_path / "m.json"))
    _, _, marg = S.posterior(cum, params)
    for b, L in enumerate(lengths):
        np.testing.assert_allclose(np.array(m["position_marginals"][b]), marg.position_marginals[b, :L], atol=1e-12)


@pytest.mark.gpu
def test_cli_bench_csv(tmp_path):
    """bench --format csv (cli.py:42-53, 131-200): the reference's columns first, then the
    fwd+bwd throughput and device peak; one row per T."""
    from paper_2604_18780_b200 import cli

    out = tmp_path / "b.csv"
    rc = cli.main(["bench", "--T", "200", "400", "--K", "20", "--C", "4", "--B", "2", "--repeats", "1",
                   "--format", "csv", "--out", str(out)])
    assert rc == 0
    lines = out.read_text().strip().splitlines()
    assert lines[0].startswith("#")
    header = lines[1].split(",")
    assert header[: len(cli.BENCH_COLUMNS)] == list(cli.BENCH_COLUMNS)
    assert len(lines) == 4
    for row in lines[2:]:
        cells = dict(zip(header, row.split(",")))
        assert cells["status"] == "ok" and float(cells["positions_per_sec_fwd_bwd"]) > 0
