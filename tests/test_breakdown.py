"""Measured six-category breakdown (breakdown.py): charging rules and the
reference's CSV formats (simulator.py:529-544,673-704)."""
import pytest

from paper_2107_06533_b200 import breakdown as BD


def _ev(s, e, name, stream=1):
    return (s, e, name, stream)


def test_categories_partition_span_and_comm_counts_only_exposed():
    ks = [_ev(0, 10, "cudnn::conv_fwd", 1),                      # FFBP
          _ev(2, 6, "void spd::stage_rows_kernel<1>(x)", 2),      # FactorComp (overlapped by FFBP)
          _ev(8, 14, "ncclDevKernel_AllReduce_Sum_f32", 3),        # FactorComm: 10..14 exposed
          _ev(14, 16, "spd::pivot_kernel(x)", 4),                  # InverseComp
          _ev(17, 20, "ncclDevKernel_Broadcast", 3),               # InverseComm (idle 16..17)
          _ev(20, 22, "void spd::tc3_gemm_kernel<(spd::Kind)2, 3, false, 4>(x)", 1)]  # Precondition
    lab = BD.label_events(ks, ["factor", "inverse"])
    cats = [c for *_, c in lab]
    assert cats == ["FFBP", "FactorComp", "FactorComm", "InverseComp", "InverseComm", "Precondition"]
    tot = BD.breakdown(lab)
    assert tot["FFBP"] == 10 and tot["FactorComp"] == 0 and tot["FactorComm"] == 4
    assert tot["InverseComp"] == 2 and tot["Idle"] == 1 and tot["InverseComm"] == 3 and tot["Precondition"] == 2
    assert sum(tot.values()) == 22


def test_factor_syrk_off_main_stream_is_factor_comp():
    ks = [_ev(0, 5, "cutlass3x_sm100_tensorop_fprop", 7),
          _ev(1, 3, "void spd::tc3_gemm_kernel<(spd::Kind)1, 3, false, 0>(x)", 9),
          _ev(6, 7, "void spd::tc3_pair_kernel<3>(x)", 9),
          _ev(7, 9, "void spd::tc3_gemm_kernel<(spd::Kind)2, 3, true, 0>(x)", 9)]
    tot = BD.breakdown(BD.label_events(ks, []))
    assert tot["FFBP"] == 5 and tot["FactorComp"] == 1 and tot["InverseComp"] == 2 and tot["Idle"] == 1


def test_grad_tag_and_tag_count_mismatch():
    ks = [_ev(0, 1, "ncclDevKernel_AllReduce", 3), _ev(1, 2, "ncclDevKernel_AllReduce", 3)]
    lab = BD.label_events(ks, ["factor", "grad"])
    assert [c for *_, c in lab] == ["FactorComm", "GradComm"]
    with pytest.raises(ValueError):
        BD.label_events(ks, ["factor"])


def test_csv_formats_match_reference():
    csv = BD.breakdown_to_csv({"FFBP": 0.5, "GradComm": 0.25}, extra=False)
    assert csv.splitlines() == ["category,seconds", "FFBP,0.500000000", "GradComm,0.250000000",
                                "FactorComp,0.000000000", "FactorComm,0.000000000", "InverseComp,0.000000000",
                                "InverseComm,0.000000000"]
    tl = BD.timeline_to_csv([(1.0, 2.0, "k", 5, "FactorComm")], t0=1.0).splitlines()
    assert tl[0] == "event,category,resource,start,end,layer"
    assert tl[1] == "k,FactorComm,comm,0.000000000,1.000000000,stream5"


def test_classify_kernel_names():
    """Kernel-name rules of the current library (precondition = TF32 engine with chunked accumulation)."""
    from paper_2107_06533_b200.breakdown import classify
    assert classify("void spd::tc3_gemm_kernel<(spd::Kind)1, 3, false, 0>(...)") == "FactorComp"
    assert classify("void spd::tc3_pair_kernel<3>(...)") == "FactorComp"
    assert classify("void spd::stage_packed_kernel<false>(spd::StagePackedArgs)") == "Precondition"
    assert classify("spd::peer_wait_kernel(const int *, int, int, int, const int *, int *, unsigned long)") == "FactorComm"
    assert classify("spd::peer_sum_kernel(float *, const float *, long, int, int, const spd::PeerSeg *)") == "FactorComm"
    assert classify("void spd::tc3_gemm_kernel<(spd::Kind)2, 3, false, 4>(...)") == "Precondition"
    assert classify("void spd::tc3_gemm_kernel<(spd::Kind)2, 3, true, 0>(...)") == "InverseComp"
    assert classify("void spd::tc3_gemm_kernel<(spd::Kind)2, 3, false, 0>(...)") == "InverseComp"
    assert classify("void spd::pivot_tc_kernel<false>(...)") == "InverseComp"
    assert classify("void spd::tc3_gemm_kernel<(spd::Kind)0, 3, true, 0, false>(...)") == "InverseComp"  # fp16 planes
    assert classify("void spd::tc3_gemm_kernel<(spd::Kind)0, 3, false, 0, false>(...)") == "InverseComp"
    assert classify("void spd::pivot_kernel<true>(...)") == "InverseComp"
    assert classify("spd::inv_scale_kernel(...)") == "InverseComp"
    assert classify("sm100_xmma_fprop_implicit_gemm") == "FFBP"
