"""Host-format colourings through the C ABI (plse_set_colors / plse_get_colors): u16 rows [p, |V|] are
narrowed to the device's u8 rows and checked against the vertex domains on the device (every colour 0 or
not prefilled in its row or column, lsgraph.hpp:152-156); an invalid colouring is refused with the
same error as before and leaves the target buffer as it was."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,r,s,p", [(20, 0.5, 3, 40), (60, 0.5, 12345, 256), (70, 0.6, 12345, 96)])
def test_round_trip_and_domain_check(plse, orc, n, r, s, p):
    grid = orc.generate_instance(n, r, s)
    g = plse.preprocess(grid)
    pop = plse.DevicePopulation(g, plse.SolverConfig(p=p, master_seed=3))
    init = orc.init_population(grid, p, 3)
    rng = np.random.default_rng(s)
    cols = init.copy()
    cols[rng.random(cols.shape) < 0.25] = 0  # uncoloured cells are in every domain
    for which in (plse.MEMBERS, plse.OFFSPRING, plse.IMPROVED):
        pop.write_colors(which, cols)
        out = np.full((p, g.vertex_count), 0xFFFF, np.uint16)
        assert pop.read_colors(which, out) is out
        assert np.array_equal(out, cols)
    f, c, _ = pop.stats(plse.MEMBERS)  # the members upload evaluates f and c on the device
    for i in range(0, p, max(1, p // 8)):
        assert (int(f[i]), int(c[i])) == orc.eval(grid, cols[i]), i
    # a colour prefilled in the vertex's row: refused, target unchanged
    v = int(np.argmax([any(grid.reshape(n, n)[int(g.cell_row[u])]) for u in range(g.vertex_count)]))
    taken = [int(x) for x in grid.reshape(n, n)[int(g.cell_row[v])] if x]
    assert taken
    bad = cols.copy()
    bad[p // 2, v] = taken[0]
    with pytest.raises(ValueError, match="assignment leaves vertex domain"):
        pop.write_colors(plse.OFFSPRING, bad)
    assert np.array_equal(pop.read_colors(plse.OFFSPRING), cols)
    too_big = cols.copy()
    too_big[-1, -1] = n + 1
    with pytest.raises(ValueError, match="assignment leaves vertex domain"):
        pop.write_colors(plse.MEMBERS, too_big)
    assert np.array_equal(pop.read_colors(plse.MEMBERS), cols)
    for i in (0, p // 3, p - 1):
        assert np.array_equal(pop.read_row(plse.MEMBERS, i), cols[i])
    with pytest.raises(ValueError, match="out of range"):
        pop.read_row(plse.MEMBERS, p)
    with pytest.raises(ValueError, match="size mismatch"):
        pop.write_colors(plse.MEMBERS, cols[:-1])
    with pytest.raises(ValueError):
        pop.read_colors(plse.MEMBERS, np.zeros((p, g.vertex_count), np.int32))
    pop.close()
