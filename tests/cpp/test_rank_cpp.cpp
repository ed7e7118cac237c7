// The multi-GPU runtime driven from C++ only (no Python): W processes, one
// rank each, through distattn::b200::RankRuntime (include/distattn/b200.hpp
// over the C ABI), exactly as a C++ host would embed it. The bootstrap
// allgather the runtime asks for is implemented here over a shared-memory
// region (any transport works: MPI_Allgather, a TCP store, ...). The ranks
// share one GPU (the IPC transport), run the balanced forward and backward
// with the even-P split, and each checks its chunk of O / LSE / dQ / dK / dV against the C
// oracle's stepper executors (the bit-exact restatement of the reference).
//
//   tests/cpp/_build/test_rank_cpp [world] [n] [heads]
// Built by __graft_entry__.build(); run by tests/test_cpp_api.py (GPU).
#include <sys/mman.h>
#include <sys/wait.h>
#include <unistd.h>

#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "distattn/b200.hpp"
#include "distattn_oracle.h"

namespace b2 = distattn::b200;

namespace {

constexpr int kMaxWorld = 16;
constexpr size_t kSlot = 1 << 16;  // bytes per rank per allgather call

// Allgather over MAP_SHARED memory: call c of every rank writes its bytes
// into slot[c % 2][rank], publishes count[rank] = c + 1 and waits until every
// rank has published call c. A rank can be at most one call ahead, so slot
// c % 2 is not rewritten before every rank has copied call c out of it.
struct Shared {
  std::atomic<int> count[kMaxWorld];
  char slot[2][kMaxWorld][kSlot];
};

struct Ctx {
  Shared* sh;
  int rank, world, calls;
};

int shm_allgather(void* ctx, const void* send, uint64_t bytes, void* recv) {
  Ctx* c = static_cast<Ctx*>(ctx);
  if (bytes > kSlot) return 1;
  const int call = c->calls++;
  std::memcpy(c->sh->slot[call % 2][c->rank], send, bytes);
  c->sh->count[c->rank].store(call + 1, std::memory_order_release);
  for (int r = 0; r < c->world; ++r)
    while (c->sh->count[r].load(std::memory_order_acquire) < call + 1) usleep(10);
  for (int r = 0; r < c->world; ++r)
    std::memcpy(static_cast<char*>(recv) + r * bytes, c->sh->slot[call % 2][r], bytes);
  return 0;
}

uint16_t to_bf16(double x) {  // x is bf16-representable (dao_make_inputs bf16=1)
  const float f = static_cast<float>(x);
  uint32_t u;
  std::memcpy(&u, &f, 4);
  return static_cast<uint16_t>(u >> 16);
}

double from_bf16(uint16_t b) {
  const uint32_t u = static_cast<uint32_t>(b) << 16;
  float f;
  std::memcpy(&f, &u, 4);
  return f;
}

double rel(const std::vector<double>& a, const std::vector<double>& b) {
  double e = 0, m = 1e-30;
  for (size_t i = 0; i < a.size(); ++i) {
    e = std::fmax(e, std::fabs(a[i] - b[i]));
    m = std::fmax(m, std::fabs(b[i]));
  }
  return e / m;
}

int run_rank(Shared* sh, int rank, int world, int64_t n, int heads) {
  const int64_t d = 128, rows = n / world;
  Ctx ctx{sh, rank, world, 0};
  if (cudaSetDevice(0) != cudaSuccess) return 10;
  cudaStream_t st;
  cudaStreamCreate(&st);
  std::vector<double> q(heads * n * d), k(q.size()), v(q.size()), g(q.size());
  dao_make_inputs(0, world, n, d, heads, 1, q.data(), k.data(), v.data(), g.data());
  // this rank's chunk, [heads][rows][128] bf16
  auto shard = [&](const std::vector<double>& full) {
    std::vector<uint16_t> s(heads * rows * d);
    for (int h = 0; h < heads; ++h)
      for (int64_t r = 0; r < rows; ++r)
        for (int64_t c = 0; c < d; ++c)
          s[(h * rows + r) * d + c] = to_bf16(full[(h * n + rank * rows + r) * d + c]);
    return s;
  };
  b2::DeviceBuffer<uint16_t> dq_in(heads * rows * d), dk_in(dq_in.size()), dv_in(dq_in.size()),
      dg_in(dq_in.size()), out(dq_in.size());
  b2::DeviceBuffer<float> lse(heads * rows), dq(dq_in.size()), dk(dq_in.size()), dv(dq_in.size());
  const auto hq = shard(q), hk = shard(k), hv = shard(v), hg = shard(g);
  dq_in.upload(hq.data(), st);
  dk_in.upload(hk.data(), st);
  dv_in.upload(hv.data(), st);
  dg_in.upload(hg.data(), st);
  int status = 0;
  try {
    da_rank_options opts{DA_TRANSPORT_IPC, /*deterministic=*/1, 0};
    b2::RankRuntime rt(rank, world, shm_allgather, &ctx, opts);
    const b2::Chunk cq{dq_in.data(), heads, rows}, ck{dk_in.data(), heads, rows},
        cv{dv_in.data(), heads, rows};
    rt.forward(cq, ck, cv, out.data(), lse.data(), DA_SCHEDULE_BALANCED_SPLIT, st);
    rt.backward(dg_in.data(), dq.data(), dk.data(), dv.data(), DA_SCHEDULE_BALANCED_SPLIT_BWD, st);
    const auto o16 = out.download(st);
    const auto l = lse.download(st), gq = dq.download(st), gk = dk.download(st),
               gv = dv.download(st);
    for (int h = 0; h < heads && status == 0; ++h) {
      const size_t off = static_cast<size_t>(h) * n * d;
      std::vector<double> o_r(n * d), l_r(n), rq(n * d), rk(n * d), rv(n * d);
      int64_t c10[10];
      dao_run_forward(world, 4, n, d, q.data() + off, k.data() + off, v.data() + off, o_r.data(),
                      l_r.data(), c10);
      dao_run_backward_sched(world, 4, n, d, q.data() + off, k.data() + off, v.data() + off,
                             o_r.data(), l_r.data(), g.data() + off, rq.data(), rk.data(),
                             rv.data(), c10);
      std::vector<double> go, gr, qq, qr, kk, kr, vv, vr;
      double lerr = 0;
      for (int64_t r = 0; r < rows; ++r) {
        const int64_t row = rank * rows + r;
        lerr = std::fmax(lerr, std::fabs(l[h * rows + r] - l_r[row]));
        for (int64_t c = 0; c < d; ++c) {
          const size_t mine = (h * rows + r) * d + c, ref = row * d + c;
          go.push_back(from_bf16(o16[mine]));
          gr.push_back(o_r[ref]);
          qq.push_back(gq[mine]);
          qr.push_back(rq[ref]);
          kk.push_back(gk[mine]);
          kr.push_back(rk[ref]);
          vv.push_back(gv[mine]);
          vr.push_back(rv[ref]);
        }
      }
      const double eo = rel(go, gr), eq = rel(qq, qr), ek = rel(kk, kr), ev = rel(vv, vr);
      std::printf("rank %d head %d: O %.2e LSE %.2e dQ %.2e dK %.2e dV %.2e\n", rank, h, eo, lerr,
                  eq, ek, ev);
      if (!(eo < 2e-2 && lerr < 1e-3 && eq < 2e-2 && ek < 2e-2 && ev < 2e-2)) status = 2;
    }
    // deterministic runtime: a second pass repeats every bit
    rt.forward(cq, ck, cv, out.data(), lse.data(), DA_SCHEDULE_BALANCED_SPLIT, st);
    rt.backward(dg_in.data(), dq.data(), dk.data(), dv.data(), DA_SCHEDULE_BALANCED_SPLIT_BWD, st);
    if (dq.download(st) != gq || dk.download(st) != gk || out.download(st) != o16) status = 3;
  } catch (const std::exception& e) {
    std::printf("rank %d: %s\n", rank, e.what());
    status = 4;
  }
  return status;
}

}  // namespace

int main(int argc, char** argv) {
  const int world = argc > 1 ? std::atoi(argv[1]) : 4;
  const int64_t n = argc > 2 ? std::atoll(argv[2]) : 2048;
  const int heads = argc > 3 ? std::atoi(argv[3]) : 2;
  if (world < 1 || world > kMaxWorld || n % world != 0) return 2;
  void* mem = mmap(nullptr, sizeof(Shared), PROT_READ | PROT_WRITE, MAP_SHARED | MAP_ANONYMOUS,
                   -1, 0);
  if (mem == MAP_FAILED) return 2;
  Shared* sh = new (mem) Shared();
  for (auto& c : sh->count) c.store(0);
  std::vector<pid_t> kids;
  for (int r = 0; r < world; ++r) {  // CUDA is first touched in the children
    const pid_t pid = fork();
    if (pid == 0) {
      const int s = run_rank(sh, r, world, n, heads);
      std::fflush(stdout);
      _exit(s);
    }
    kids.push_back(pid);
  }
  int worst = 0;
  for (pid_t pid : kids) {
    int ws = 0;
    waitpid(pid, &ws, 0);
    const int code = WIFEXITED(ws) ? WEXITSTATUS(ws) : 100;
    worst = code > worst ? code : worst;
  }
  std::printf("%s: world %d, n %lld, heads %d\n", worst == 0 ? "PASS" : "FAIL", world,
              static_cast<long long>(n), heads);
  return worst;
}
