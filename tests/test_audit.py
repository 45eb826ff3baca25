"""The write audit derived from program extents (ulv_factor.audit_writes,
reference ulv_factor.py:50-67, 319-337): CPU checks on synthetic slab
regions, including deliberately bad programs."""
from paper_2502_02395_b200.ulv_factor import audit_writes

# two diag boxes (n = 8, r = 5) and one off-diagonal pair (8 x 8, r_i = 5, r_j = 5), 8-byte doubles
H0, H1, T = 1000, 1000 + 8 * 64, 9000
REGIONS = [(H0, 8, 8, 5, 5, ("diag", 1, 0, 0)), (H1, 8, 8, 5, 5, ("diag", 1, 1, 1)),
           (T, 8, 8, 5, 5, ("off", 1, 1, 0))]


def good_program():
    w = []
    for h in (H0, H1):
        w.append((0, "transform", h, 8, 8, 8, True))              # H = Q^T A Q (lower)
        w.append((1, "factor", h, 8, 5, 8, False))                # panel: columns 0..4, all rows
        w.append((2, "factor", h + 8 * (2 * 8 + 2), 6, 3, 8, True))   # REST: RR columns 2..4 + SR rows
        w.append((3, "schur", h + 8 * (5 * 8 + 5), 3, 3, 8, True))    # SS -= L(s) L(s)^T
    w.append((4, "transform", T + 8 * (5 * 8 + 5), 3, 3, 8, False))   # SS_ij (lane 2)
    w.append((5, "transform", T, 8, 5, 8, False))                     # T[:, :r_j] (lane 3)
    w.append((6, "merge", 50000, 6, 6, 6, False))                     # parent block: not a slab
    return w


def test_clean_program_matches_reference_contract():
    a = audit_writes(REGIONS, good_program())
    assert a["offdiag_ss_post_init_writes"] == 0 and a["rr_rs_sr_post_init_writes"] == 0
    assert a["diag_ss_update_counts"] == [1] and a["diag_ss_blocks"] == 2
    assert a["in_place_factor_writes"] == 8 and a["uninitialized_slabs"] == 0 and a["initialized_twice"] == 0


def test_bad_programs_are_caught():
    w = good_program() + [(7, None, T + 8 * (6 * 8 + 6), 1, 1, 8, False)]      # stray write into SS_ij
    assert audit_writes(REGIONS, w)["offdiag_ss_post_init_writes"] == 1
    w = good_program() + [(7, "schur", H0 + 8 * (5 * 8 + 5), 3, 3, 8, True)]   # second Schur update
    assert audit_writes(REGIONS, w)["diag_ss_update_counts"] == [1, 2]
    w = good_program() + [(7, "factor", T, 2, 2, 8, False)]                     # "factor" write into lr_off
    assert audit_writes(REGIONS, w)["rr_rs_sr_post_init_writes"] == 1
    w = good_program() + [(7, "factor", H1 + 8 * (6 * 8 + 5), 1, 2, 8, False)]  # factor write spilling into SS
    assert audit_writes(REGIONS, w)["diag_ss_update_counts"] == [1, 2]
    w = [x for x in good_program() if x[0] != 4]                                # SS_ij never formed
    assert audit_writes(REGIONS, w)["uninitialized_slabs"] == 1
    w = good_program() + [(8, "transform", T, 8, 5, 8, False)]                  # formed twice
    assert audit_writes(REGIONS, w)["initialized_twice"] == 2


def test_vacuous_schur_of_full_rank_box_counts_once():
    regions = [(H0, 8, 8, 0, 0, ("diag", 1, 0, 0))]                  # r = 0: nothing to eliminate
    a = audit_writes(regions, [(0, "transform", H0, 8, 8, 8, True)])
    assert a["diag_ss_update_counts"] == [1]


def test_edge_carved_transform_counts_once():
    """A transform stored by disjoint pieces (Program.gemm carves the ragged edge strips
    of a plain problem into the 32x32-tile launch) initializes each slab once; pieces
    that overlap are still an initialization twice."""
    w = [x for x in good_program() if x[0] != 5]
    carved = w + [(5, "transform", T, 4, 5, 8, False),                    # rows 0..3 of T[:, :r_j]
                  (9, "transform", T + 8 * (4 * 8), 4, 5, 8, False)]      # rows 4..7: the edge strip
    a = audit_writes(REGIONS, carved)
    assert a["initialized_twice"] == 0 and a["uninitialized_slabs"] == 0
    overlap = w + [(5, "transform", T, 5, 5, 8, False), (9, "transform", T + 8 * (4 * 8), 4, 5, 8, False)]
    assert audit_writes(REGIONS, overlap)["initialized_twice"] == 1
