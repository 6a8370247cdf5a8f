"""Host-side configuration objects (no GPU)."""

def test_mgconfig_coarse_solver_validation():
    import pytest

    from paper_2603_28706_b200.stmg import MgConfig

    assert MgConfig().coarse_solver == "dense"  # the reference's coarse LU by default
    MgConfig(coarse_solver="vanka", coarse_sweeps=0, coarse_omega=1.0)
    for bad in (dict(coarse_solver="lu"), dict(coarse_sweeps=-1), dict(coarse_omega=0.0), dict(coarse_omega=1.5)):
        with pytest.raises(ValueError):
            MgConfig(**bad)
