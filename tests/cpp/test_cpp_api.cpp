// C++ drop-in check: the reference's DipoleTree usage pattern, compiled against
// include/dipole_b200.hpp (the C++ mirror over the C-ABI) and checked against
// the CPU oracle (oracle/dipole_oracle.h — test infrastructure only). Mirrors
// cases of proj/tests/test_bhtree.cpp with fp32 tolerances. Exit code 0 = pass.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <random>
#include <vector>

#include "../../include/dipole_b200.hpp"
extern "C" {
#include "../../oracle/dipole_oracle.h"
}

using namespace dipole_b200;

static int failures = 0;
#define EXPECT(cond)                                                        \
  do {                                                                      \
    if (!(cond)) {                                                          \
      ++failures;                                                           \
      std::fprintf(stderr, "%s:%d: EXPECT(%s) failed\n", __FILE__, __LINE__, #cond); \
    }                                                                       \
  } while (0)

static PointCloud random_cloud(int n, unsigned seed, int C) {
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> uni(-1.0, 1.0);
  std::normal_distribution<double> gauss(0.0, 1.0);
  PointCloud c;
  c.channels = C;
  for (int i = 0; i < n; ++i) {
    for (int a = 0; a < 3; ++a) c.positions.push_back((double)(float)uni(rng));
    double v[3] = {gauss(rng), gauss(rng), gauss(rng)};
    double l = std::sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
    for (int a = 0; a < 3; ++a) c.normals.push_back(v[a] / l);
    c.areas.push_back((0.5 + 0.5 * std::fabs(uni(rng))) / n);
    for (int k = 0; k < C; ++k) c.moments.push_back(uni(rng));
  }
  return c;
}

int main() {
  // degenerate builds (test_bhtree.cpp:28-61)
  {
    DipoleTree t;
    PointCloud one;
    one.positions = {1, 2, 3};
    one.normals = {0, 0, 1};
    one.areas = {0.7};
    one.moments = {1.0};
    t.build(one);
    auto nd = t.nodes();
    EXPECT(nd.size() == 1 && nd[0].leaf && nd[0].area == 0.7 && nd[0].radius == 0.0);
    PointCloud two = one;
    two.positions.insert(two.positions.end(), {3, 2, 3});
    two.normals.insert(two.normals.end(), {0, 0, 1});
    two.areas.push_back(0.7);
    two.moments.push_back(1.0);
    t.build(two);
    nd = t.nodes();
    EXPECT(std::fabs(nd[0].centroid[0] - 2) <= 1e-15 && nd[0].centroid[1] == 2);
    bool threw = false;
    try {
      t.build(PointCloud{});
    } catch (const DataError&) {
      threw = true;
    }
    EXPECT(threw);
  }
  // random cloud: structure, forward, primal_channel, adjoint + flush vs oracle
  {
    const int n = 3000, C = 3, q = 1000;
    PointCloud c = random_cloud(n, 12, C);
    DipoleTree t;
    t.build(c);
    t.set_channel_kernels({ChannelKernel::Dipole, ChannelKernel::Radial, ChannelKernel::Radial});
    ora_tree* r = ora_tree_build(c.positions.data(), c.normals.data(), c.areas.data(),
                                 c.moments.data(), n, C, 8, 20);
    uint8_t kinds[3] = {0, 1, 1};
    ora_tree_set_kinds(r, kinds, C);
    const int64_t nn = ora_tree_node_count(r);
    std::vector<int32_t> topo(nn * 6), order(n);
    ora_tree_export(r, nullptr, topo.data(), order.data(), nullptr);
    auto nodes = t.nodes();
    EXPECT((int64_t)nodes.size() == nn);
    bool same = (int64_t)nodes.size() == nn;
    for (int64_t i = 0; same && i < nn; ++i)
      same = nodes[i].begin == topo[6 * i] && nodes[i].end == topo[6 * i + 1] &&
             nodes[i].child_begin == topo[6 * i + 2] && nodes[i].child_count == topo[6 * i + 3] &&
             nodes[i].parent == topo[6 * i + 4] && nodes[i].leaf == (topo[6 * i + 5] != 0);
    EXPECT(same);
    EXPECT(t.point_order() == std::vector<int>(order.begin(), order.end()));

    std::mt19937_64 rng(13);
    std::uniform_real_distribution<double> uni(-1.5, 1.5);
    std::vector<double> xs(3 * q);
    for (double& v : xs) v = uni(rng);
    KernelParams p;
    p.epsilon = 0.1;
    ora_params op = {0.1, 0, 0, 0.0, 0.0};
    std::vector<float> out(q * C);
    t.primal(xs.data(), q, p, 2.0, out.data());
    std::vector<double> want(q * C);
    ora_primal(r, &op, 2.0, xs.data(), q, 0, 0, want.data(), nullptr, nullptr, 4);
    int bad = 0;
    for (int i = 0; i < q * C; ++i)
      bad += std::fabs(out[i] - want[i]) > 1e-6 + 1e-4 * std::fabs(want[i]);
    EXPECT(bad == 0);
    for (int ch = 0; ch < C; ++ch) {  // primal_channel == primal()[c] (test_bhtree.cpp:140)
      std::vector<float> pc(q);
      t.primal_channel(xs.data(), q, p, 2.0, ch, pc.data());
      bool eq = true;
      for (int i = 0; i < q; ++i) eq = eq && pc[i] == out[i * C + ch];
      EXPECT(eq);
    }
    std::vector<float> d_out(q * C);
    std::normal_distribution<double> g(0, 1);
    for (float& v : d_out) v = (float)g(rng);
    std::vector<double> d_out64(d_out.begin(), d_out.end());
    GradientBuffer buf = t.make_buffer();
    t.adjoint(xs.data(), q, p, 2.0, d_out.data(), nullptr, buf);
    PointGradients pg = t.flush_gradients(buf);
    std::vector<double> wm(n * C), wn(n * 3);
    double we = 0;
    ora_adjoint(r, &op, 2.0, xs.data(), q, d_out64.data(), nullptr, 4, wm.data(), wn.data(), &we);
    double scale = 0, err = 0;
    for (int i = 0; i < n * C; ++i) {
      scale = std::fmax(scale, std::fabs(wm[i]));
      err = std::fmax(err, std::fabs(pg.moments[i] - wm[i]));
    }
    EXPECT(err <= 1e-5 * scale);
    EXPECT(std::fabs(pg.d_epsilon - we) <= 1e-4 * std::fabs(we) + 1e-6);
    // DPLT dump: header + structure bytes (bhtree.cpp:465-494)
    const char* path = "/tmp/dpl_cpp_test.dplt";
    t.dump(path);
    std::ifstream in(path, std::ios::binary);
    char magic[4];
    uint32_t ver = 0, ch = 0;
    uint64_t pts = 0, cnt = 0;
    in.read(magic, 4);
    in.read((char*)&ver, 4);
    in.read((char*)&ch, 4);
    in.read((char*)&pts, 8);
    in.read((char*)&cnt, 8);
    EXPECT(std::memcmp(magic, "DPLT", 4) == 0 && ver == 1 && ch == (uint32_t)C &&
           pts == (uint64_t)n && cnt == (uint64_t)nn);
    std::remove(path);
    bool threw = false;
    try {
      t.set_channel_kernels({ChannelKernel::Dipole});
    } catch (const DataError&) {
      threw = true;
    }
    EXPECT(threw);
    ora_tree_free(r);
  }
  std::printf("cpp api test: %s (%d failures)\n", failures ? "FAILED" : "passed", failures);
  return failures ? 1 : 0;
}
