// C++ parity tests of the drop-in API (include/distattn/b200.hpp), written
// like the reference's own suites (/root/reference/proj/tests/test_*.cpp):
// schedules field-exact against the C oracle (itself bit-exact with the
// reference build), the exception taxonomy, and on a B200 the distributed
// forward/backward against the oracle's stepper executors.
//
//   tests/cpp/_build/test_b200_api [--cpu-only]
// Built by __graft_entry__.build(); run by tests/test_cpp_api.py.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <string>
#include <vector>

#include "distattn/b200.hpp"
#include "distattn_oracle.h"

namespace b2 = distattn::b200;

static int g_pass = 0, g_fail = 0;

static void run(const char* name, const std::function<void()>& fn) {
  try {
    fn();
    ++g_pass;
    std::printf("PASS %s\n", name);
  } catch (const std::exception& e) {
    ++g_fail;
    std::printf("FAIL %s: %s\n", name, e.what());
  }
}

#define REQUIRE(c)                                                                          \
  do {                                                                                      \
    if (!(c)) throw std::runtime_error(std::string("requirement failed: ") + #c + " @" +    \
                                       std::to_string(__LINE__));                           \
  } while (0)

template <typename E>
static bool throws(const std::function<void()>& fn) {
  try {
    fn();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

static void oracle_flat(int P, int kind, std::vector<int32_t>& t, std::vector<int32_t>& m,
                        int32_t& steps) {
  int64_t nt = 0, nm = 0;
  dao_schedule_build(P, kind, &steps, nullptr, &nt, nullptr, &nm);
  t.assign(6 * nt, 0);
  m.assign(4 * (nm > 0 ? nm : 1), 0);
  dao_schedule_build(P, kind, &steps, t.data(), &nt, m.data(), &nm);
  m.resize(4 * nm);
}

static b2::bf16_t to_bf16(double x) {  // x is already bf16-representable
  float f = static_cast<float>(x);
  uint32_t u;
  std::memcpy(&u, &f, 4);
  return static_cast<b2::bf16_t>(u >> 16);
}

static double from_bf16(b2::bf16_t b) {
  uint32_t u = static_cast<uint32_t>(b) << 16;
  float f;
  std::memcpy(&f, &u, 4);
  return f;
}

static double rel(const std::vector<double>& a, const std::vector<double>& b) {
  double num = 0, den = 0;
  for (size_t i = 0; i < a.size(); ++i) {
    num = std::fmax(num, std::fabs(a[i] - b[i]));
    den = std::fmax(den, std::fabs(b[i]));
  }
  return den > 0 ? num / den : num;
}

static void schedule_tests() {
  run("schedules field-exact vs the oracle, P = 1..16 (ring, balanced, split)", [] {
    for (int kind : {0, 1, 4})
      for (int P = 1; P <= 16; ++P) {
        const b2::Schedule s = kind == 0   ? b2::build_ring_schedule(P)
                               : kind == 1 ? b2::build_balanced_schedule(P)
                                           : b2::build_balanced_split_schedule(P);
        std::vector<int32_t> t, m, to, mo;
        int32_t steps = 0;
        b2::flatten(s, t, m);
        oracle_flat(P, kind, to, mo, steps);
        REQUIRE(steps == s.step_count());
        REQUIRE(t == to);
        REQUIRE(m == mo);
        REQUIRE(b2::validate(s).empty());
      }
  });
  run("exact counts at P = 8 (test_schedule.cpp:50-85)", [] {
    const b2::Schedule r = b2::build_ring_schedule(8);
    REQUIRE(r.step_count() == 8 && r.attention_task_count() == 36 && r.idle_slot_count() == 28);
    const b2::Schedule b = b2::build_balanced_schedule(8);
    REQUIRE(b.step_count() == 5 && b.attention_task_count() == 36 && b.idle_slot_count() == 4);
    REQUIRE(b.messages.size() == 34);
  });
  run("validator flags injected faults (test_schedule.cpp:159-199)", [] {
    b2::Schedule s = b2::build_ring_schedule(3);
    s.steps[2][2] = b2::Task{};  // drop (q3, kv1)
    const auto v = b2::validate(s);
    REQUIRE(!v.empty());
    bool found = false;
    for (const auto& e : v) found = found || e.find("never computed") != std::string::npos;
    REQUIRE(found);
  });
  run("errors: ConfigError for bad workers, ragged splits (test_runtime.cpp:57-69)", [] {
    REQUIRE(throws<b2::ConfigError>([] { b2::build_ring_schedule(0); }));
    std::vector<b2::bf16_t> z(3 * 32 * 128);
    REQUIRE(throws<b2::ConfigError>([&] { b2::make_shards(3, 32, 1, z, z, z, z, nullptr); }));
  });
}

static void gpu_tests() {
  run("device supported (sm_100)", [] { REQUIRE(da_device_supported() == 1); });
  cudaStream_t st = nullptr;
  run("finalize of an untouched accumulator throws DegenerateRowError", [] {
    auto acc = b2::AttnAccumulator::make_fresh(1, 128);
    REQUIRE(throws<b2::DegenerateRowError>([&] { b2::finalize(acc, nullptr); }));
  });
  run("block_attn_update + finalize = dense causal attention (flashcore.hpp:96-197)", [&] {
    const int64_t n = 384, d = 128;
    std::vector<double> q(n * d), k(n * d), v(n * d), o(n * d), lse(n);
    dao_make_inputs(3, 1, n, d, 1, 1, q.data(), k.data(), v.data(), nullptr);
    std::vector<b2::bf16_t> qb(n * d), kb(n * d), vb(n * d);
    for (int64_t i = 0; i < n * d; ++i) {
      qb[i] = to_bf16(q[i]);
      kb[i] = to_bf16(k[i]);
      vb[i] = to_bf16(v[i]);
    }
    b2::DeviceBuffer<b2::bf16_t> dq(n * d), dk(n * d), dv(n * d);
    dq.upload(qb.data(), st);
    dk.upload(kb.data(), st);
    dv.upload(vb.data(), st);
    const double scale = 1.0 / std::sqrt(128.0);
    auto acc = b2::block_attn_update({dq.data(), 1, n}, {dk.data(), 1, n}, {dv.data(), 1, n},
                                     b2::AttnAccumulator::make_fresh(1, n),
                                     b2::MaskMode::Diagonal, scale, st);
    b2::AttnOutput out = b2::finalize(acc, st);
    dao_dense_oracle(q.data(), k.data(), v.data(), n, n, d, 1, scale, o.data(), lse.data());
    const auto ob = out.o.download(st);
    const auto lb = out.lse.download(st);
    std::vector<double> og(n * d), lg(n);
    for (int64_t i = 0; i < n * d; ++i) og[i] = from_bf16(ob[i]);
    double lerr = 0;
    for (int64_t i = 0; i < n; ++i) lerr = std::fmax(lerr, std::fabs(lb[i] - lse[i]));
    REQUIRE(rel(og, o) < 2e-2);
    REQUIRE(lerr < 1e-3);
  });
  run("run_backward without forward state throws StateError (test_runtime.cpp:270-276)", [&] {
    std::vector<b2::bf16_t> z(2 * 256 * 128, 0);
    auto s = b2::make_shards(2, 256, 1, z, z, z, z, st);
    for (auto& x : s) x.out = b2::DeviceBuffer<b2::bf16_t>();
    REQUIRE(throws<b2::StateError>([&] { b2::run_backward(s, 1, DA_SCHEDULE_RING_BWD, st); }));
  });
  run("Schedule-object runtime + allocation-free backward_into == kind entry points", [&] {
    const int P = 4;
    const int64_t n = 1024, d = 128, H = 1;
    std::vector<double> q(H * n * d), k(H * n * d), v(H * n * d), g(H * n * d);
    dao_make_inputs(2, P, n, d, H, 1, q.data(), k.data(), v.data(), g.data());
    std::vector<b2::bf16_t> qb(q.size()), kb(q.size()), vb(q.size()), gb(q.size());
    for (size_t i = 0; i < q.size(); ++i) {
      qb[i] = to_bf16(q[i]);
      kb[i] = to_bf16(k[i]);
      vb[i] = to_bf16(v[i]);
      gb[i] = to_bf16(g[i]);
    }
    auto a = b2::make_shards(P, n, H, qb, kb, vb, gb, st);
    auto b = b2::make_shards(P, n, H, qb, kb, vb, gb, st);
    b2::run_forward(a, H, DA_SCHEDULE_BALANCED, st);
    b2::run_forward(b, H, b2::build_balanced_schedule(P), b2::RunOptions{}, st);
    for (int p = 0; p < P; ++p) {
      REQUIRE(a[p].out.download(st) == b[p].out.download(st));
      REQUIRE(a[p].lse.download(st) == b[p].lse.download(st));
    }
    REQUIRE(throws<b2::ConfigError>([&] {
      b2::RunOptions bad;
      bad.block_rows = 0;
      b2::run_forward(b, H, b2::build_ring_schedule(P), bad, st);
    }));
    // worker 1's diagonal pair through the allocation-free form, twice with one
    // workspace: deterministic dq, identical to the value form
    const b2::Chunk cq{a[0].q.data(), H, n / P}, ck{a[0].k.data(), H, n / P},
        cv{a[0].v.data(), H, n / P}, co{a[0].out.data(), H, n / P},
        cg{a[0].d_out.data(), H, n / P};
    b2::Workspace ws;
    b2::ChunkGrads into{b2::DeviceBuffer<float>(H * (n / P) * d),
                        b2::DeviceBuffer<float>(H * (n / P) * d),
                        b2::DeviceBuffer<float>(H * (n / P) * d)};
    cudaMemsetAsync(into.dq.data(), 0, into.dq.size() * 4, st);
    b2::block_attn_backward_into(cq, ck, cv, co, a[0].lse.data(), cg, b2::MaskMode::Diagonal,
                                 1.0 / std::sqrt(128.0), into, ws, st, false, true);
    const auto val = b2::block_attn_backward(cq, ck, cv, co, a[0].lse.data(), cg,
                                             b2::MaskMode::Diagonal, 1.0 / std::sqrt(128.0), st,
                                             true);
    REQUIRE(into.dq.download(st) == val.dq.download(st));
    REQUIRE(into.dk.download(st) == val.dk.download(st));
    REQUIRE(throws<b2::ShapeError>([&] {
      const b2::Chunk half{a[0].v.data(), H, n / P / 2};
      b2::block_attn_backward_into(cq, ck, half, co, a[0].lse.data(), cg, b2::MaskMode::Diagonal,
                                   1.0, into, ws, st);
    }));
  });
  for (int kind : {0, 1, 4}) {
    const std::string name = std::string("P=4 N=2048 H=2 forward (") +
                             (kind == 0 ? "ring" : kind == 1 ? "balanced" : "split") +
                             ") + " + (kind == 4 ? "split (Schedule object)" : "ring") +
                             " backward vs the oracle stepper, counters exact";
    run(name.c_str(), [&, kind] {
      const int P = 4;
      const int64_t n = 2048, d = 128, H = 2;
      std::vector<double> q(H * n * d), k(H * n * d), v(H * n * d), g(H * n * d);
      dao_make_inputs(0, P, n, d, H, 1, q.data(), k.data(), v.data(), g.data());
      std::vector<b2::bf16_t> qb(q.size()), kb(q.size()), vb(q.size()), gb(q.size());
      for (size_t i = 0; i < q.size(); ++i) {
        qb[i] = to_bf16(q[i]);
        kb[i] = to_bf16(k[i]);
        vb[i] = to_bf16(v[i]);
        gb[i] = to_bf16(g[i]);
      }
      auto shards = b2::make_shards(P, n, H, qb, kb, vb, gb, st);
      const auto cf = b2::run_forward(shards, H, static_cast<da_schedule_kind>(kind), st);
      const auto cb =
          kind == 4 ? b2::run_backward(shards, H, b2::build_balanced_split_backward_schedule(P),
                                       b2::RunOptions{}, st)
                    : b2::run_backward(shards, H, DA_SCHEDULE_RING_BWD, st);
      const int64_t rows = n / P;
      for (int64_t h = 0; h < H; ++h) {
        const size_t off = h * n * d;
        std::vector<double> o(n * d), lse(n), rq(n * d), rk(n * d), rv(n * d);
        int64_t c10[10], b10[10];
        dao_run_forward(P, kind, n, d, q.data() + off, k.data() + off, v.data() + off, o.data(),
                        lse.data(), c10);
        if (kind == 4)  // the oracle over the same split backward table
          dao_run_backward_sched(P, 4, n, d, q.data() + off, k.data() + off, v.data() + off,
                                 o.data(), lse.data(), g.data() + off, rq.data(), rk.data(),
                                 rv.data(), b10);
        else
          dao_run_backward(P, n, d, q.data() + off, k.data() + off, v.data() + off, o.data(),
                           lse.data(), g.data() + off, rq.data(), rk.data(), rv.data(), b10);
        std::vector<double> go(n * d), gl(n), gq(n * d), gk(n * d), gv(n * d);
        for (int p = 0; p < P; ++p) {
          const auto so = shards[p].out.download(st);
          const auto sl = shards[p].lse.download(st);
          const auto sq = shards[p].dq.download(st);
          const auto sk = shards[p].dk.download(st);
          const auto sv = shards[p].dv.download(st);
          for (int64_t r = 0; r < rows; ++r) {
            gl[p * rows + r] = sl[h * rows + r];
            for (int64_t c = 0; c < d; ++c) {
              const size_t src = (h * rows + r) * d + c, dst = (p * rows + r) * d + c;
              go[dst] = from_bf16(so[src]);
              gq[dst] = sq[src];
              gk[dst] = sk[src];
              gv[dst] = sv[src];
            }
          }
        }
        double lerr = 0;
        for (int64_t i = 0; i < n; ++i) lerr = std::fmax(lerr, std::fabs(gl[i] - lse[i]));
        REQUIRE(rel(go, o) < 2e-2);
        REQUIRE(lerr < 1e-3);
        REQUIRE(rel(gq, rq) < 2e-2);
        REQUIRE(rel(gk, rk) < 2e-2);
        REQUIRE(rel(gv, rv) < 2e-2);
        if (h == 0) {  // device counters are per head x H (runtime.cpp:50-83)
          REQUIRE(cf.kv_scalars == c10[0] * H && cf.q_scalars == c10[1] * H &&
                  cf.partial_scalars == c10[2] * H && cf.kv_messages == c10[4] &&
                  cf.attention_kernel_calls == c10[8]);
          REQUIRE(cb.kv_scalars == b10[0] * H && cb.grad_scalars == b10[3] * H &&
                  cb.grad_messages == b10[7] && cb.attention_kernel_calls == b10[8]);
        }
      }
    });
  }
}

int main(int argc, char** argv) {
  const bool cpu_only = argc > 1 && std::strcmp(argv[1], "--cpu-only") == 0;
  schedule_tests();
  if (!cpu_only) gpu_tests();
  std::printf("%d passed, %d failed\n", g_pass, g_fail);
  return g_fail == 0 ? 0 : 1;
}
