// Driver linked against the UNMODIFIED reference sources under
// /root/reference/proj (built by oracle/Makefile into oracle/_ref/). It is the
// parity oracle's ground truth and the CPU baseline of bench.py:
//
//   ref_driver schedules                      -> JSON: ring/balanced tables P=1..16
//   ref_driver rng                            -> JSON: splitmix64 KAT
//   ref_driver run N P H D SEED SCHED OUTDIR [bf16]
//        runs make_shards/run_forward/run_backward (reference executors),
//        writes q,k,v,d_out,out,lse,dq,dk,dv as float64 [H][N][D] binaries
//        plus counters/trace JSON. bf16=1 rounds q/k/v/d_out to bf16 first.
//   ref_driver ckpt                           -> JSON: checkpoint plans (ckptplan.cpp):
//        positions, recompute counts of run_with_checkpointing on a small
//        pipeline, cost-model times, saved scalars, cross-plan bitwise flags
//   ref_driver time N P H D SCHED THREADS
//        wall time of forward+backward with the reference's concurrent
//        executor (P threads per head; heads spread over THREADS/P workers).
//
// Test infrastructure only. Input convention (documented in DESIGN.md):
// per head h, head_rng = Rng(seed).fork() (h+1-th fork), shards =
// make_shards(P, N, D, head_rng) (q, then k, then v), then
// d_out = head_rng.matrix(N, D).
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iostream>
#include <string>
#include <thread>
#include <vector>

#include "distattn/ckptplan.hpp"
#include "distattn/flashcore.hpp"
#include "distattn/numerics.hpp"
#include "distattn/runtime.hpp"
#include "distattn/schedule.hpp"

namespace da = distattn;

static double bf16_round(double x) {
  float f = static_cast<float>(x);
  uint32_t u;
  std::memcpy(&u, &f, 4);
  const uint32_t lsb = (u >> 16) & 1u;
  u = (u + 0x7FFFu + lsb) & 0xFFFF0000u;
  std::memcpy(&f, &u, 4);
  return static_cast<double>(f);
}

static void round_mat(da::Matd& m) {
  for (da::Index i = 0; i < m.rows(); ++i)
    for (da::Index j = 0; j < m.cols(); ++j) m(i, j) = bf16_round(m(i, j));
}

static void dump_schedule(std::ostream& os, const da::Schedule& s) {
  os << "{\"P\":" << s.workers << ",\"steps\":" << s.step_count() << ",\"tasks\":[";
  bool first = true;
  for (size_t t = 0; t < s.steps.size(); ++t)
    for (const auto& k : s.steps[t]) {
      os << (first ? "" : ",") << "[" << t << "," << static_cast<int>(k.kind) << "," << k.worker
         << "," << k.query_owner << "," << k.kv_owner << "," << k.helper << "]";
      first = false;
    }
  os << "],\"messages\":[";
  first = true;
  for (const auto& m : s.messages) {
    os << (first ? "" : ",") << "[" << m.step << "," << m.from << "," << m.to << ","
       << static_cast<int>(m.kind) << "]";
    first = false;
  }
  const auto idle = da::idle_fraction(s);
  const auto sp = da::expected_speedup(s);
  os << "],\"attention\":" << s.attention_task_count() << ",\"idle\":" << s.idle_slot_count()
     << ",\"merges\":" << s.merge_count() << ",\"idle_fraction\":[" << idle.num() << ","
     << idle.den() << "],\"speedup\":[" << sp.num() << "," << sp.den()
     << "],\"violations\":" << da::validate(s).size() << "}";
}

static void write_bin(const std::string& path, const std::vector<double>& v) {
  std::ofstream f(path, std::ios::binary);
  f.write(reinterpret_cast<const char*>(v.data()), static_cast<std::streamsize>(v.size() * 8));
}

struct HeadData {
  std::vector<da::SequenceShard> shards;
};

static std::vector<da::SequenceShard> make_head(int P, da::Index N, da::Index D, da::Rng& rng,
                                                bool bf16) {
  da::Rng head_rng = rng.fork();
  auto shards = da::make_shards(P, N, D, head_rng);
  const da::Matd dout = head_rng.matrix(N, D);
  const da::Index rows = N / P;
  for (int p = 0; p < P; ++p) {
    shards[p].d_out = dout.middleRows(p * rows, rows);
    if (bf16) {
      round_mat(shards[p].q);
      round_mat(shards[p].k);
      round_mat(shards[p].v);
      round_mat(shards[p].d_out);
    }
  }
  return shards;
}

static da::Schedule pick(const std::string& s, int P) {
  return s == "ring" ? da::build_ring_schedule(P) : da::build_balanced_schedule(P);
}

int main(int argc, char** argv) {
  if (argc < 2) {
    std::cerr << "usage: ref_driver schedules|rng|run|time ...\n";
    return 2;
  }
  const std::string mode = argv[1];
  try {
    if (mode == "schedules") {
      std::cout << "{\"ring\":[";
      for (int P = 1; P <= 16; ++P) {
        if (P > 1) std::cout << ",";
        dump_schedule(std::cout, da::build_ring_schedule(P));
      }
      std::cout << "],\"balanced\":[";
      for (int P = 1; P <= 16; ++P) {
        if (P > 1) std::cout << ",";
        dump_schedule(std::cout, da::build_balanced_schedule(P));
      }
      std::cout << "]}\n";
      return 0;
    }
    if (mode == "ckpt") {
      const da::CheckpointStrategy strats[3] = {da::CheckpointStrategy::None,
                                                 da::CheckpointStrategy::LayerBoundary,
                                                 da::CheckpointStrategy::AttentionOutput};
      const da::CkptCostModel cost{3.0, 5.0, 11.0};
      std::cout << "{\"cases\":[";
      bool first = true;
      for (int L = 1; L <= 3; ++L) {
        const da::LayerPipeline pipe = da::make_pipeline(L, 12, 4, 8, 7);
        da::Rng r(11);
        const da::Matd x = r.matrix(12, 4, -1.0, 1.0);
        const da::Matd g = r.matrix(12, 4, -1.0, 1.0);
        std::vector<da::CkptRunResult> runs;
        for (const auto st : strats) {
          const da::CheckpointPlan pl = da::plan(pipe, st);
          runs.push_back(da::run_with_checkpointing(pipe, pl, x, g));
          const auto& tr = runs.back().trace;
          std::cout << (first ? "" : ",") << "{\"layers\":" << L << ",\"strategy\":\""
                    << da::to_string(st) << "\",\"positions\":[";
          for (size_t i = 0; i < pl.saved_positions.size(); ++i)
            std::cout << (i ? "," : "") << pl.saved_positions[i];
          std::cout << "],\"counts\":[";
          for (int k = 0; k < da::kOpsPerLayer; ++k) std::cout << (k ? "," : "") << tr.counts[k];
          std::cout << "],\"iteration_time\":" << da::iteration_time_model(cost, L, st)
                    << ",\"recompute_time\":" << da::recompute_time(tr, cost)
                    << ",\"saved_activation_scalars\":" << da::saved_activation_scalars(pl, pipe)
                    << "}";
          first = false;
        }
        // the reference's bitwise cross-plan property (ckptplan.hpp:8-9)
        for (size_t i = 1; i < runs.size(); ++i) {
          const auto& a = runs[0].grads;
          const auto& b = runs[i].grads;
          bool same = true;
          for (da::Index j = 0; j < a.d_input.size(); ++j)
            same = same && a.d_input.data()[j] == b.d_input.data()[j];
          if (!same) throw std::runtime_error("reference cross-plan grads differ");
        }
      }
      std::cout << "],\"cost\":[3.0,5.0,11.0]}\n";
      return 0;
    }
    if (mode == "ckpt128") {
      // the checkpointed layer pipeline at the kernels' head dim (d = 128,
      // 256 tokens): the three plans' input gradients must be bit-identical
      // (ckptplan.hpp:8-9); the first plan's d_input is written to OUT.
      if (argc < 3) throw da::ConfigError("ckpt128 OUT");
      const da::CheckpointStrategy strats[3] = {da::CheckpointStrategy::None,
                                                 da::CheckpointStrategy::LayerBoundary,
                                                 da::CheckpointStrategy::AttentionOutput};
      const da::LayerPipeline pipe = da::make_pipeline(2, 256, 128, 256, 7);
      da::Rng r(11);
      const da::Matd x = r.matrix(256, 128, -1.0, 1.0);
      const da::Matd g = r.matrix(256, 128, -1.0, 1.0);
      std::vector<da::CkptRunResult> runs;
      std::cout << "{\"counts\":[";
      for (int i = 0; i < 3; ++i) {
        runs.push_back(da::run_with_checkpointing(pipe, da::plan(pipe, strats[i]), x, g));
        std::cout << (i ? "," : "") << "[";
        for (int k = 0; k < da::kOpsPerLayer; ++k)
          std::cout << (k ? "," : "") << runs.back().trace.counts[k];
        std::cout << "]";
      }
      bool same = true;
      for (size_t i = 1; i < runs.size(); ++i)
        for (da::Index j = 0; j < runs[0].grads.d_input.size(); ++j)
          same = same && runs[0].grads.d_input.data()[j] == runs[i].grads.d_input.data()[j];
      std::vector<double> dx(runs[0].grads.d_input.data(),
                             runs[0].grads.d_input.data() + runs[0].grads.d_input.size());
      write_bin(argv[2], dx);
      std::cout << "],\"bitwise_equal\":" << (same ? "true" : "false") << "}\n";
      return 0;
    }
    if (mode == "rng") {
      da::Rng r(0);
      std::cout << "{\"seed0_u64\":[";
      for (int i = 0; i < 8; ++i) std::cout << (i ? "," : "") << "\"" << r.next_u64() << "\"";
      da::Rng r2(12345);
      std::cout << "],\"seed12345_unit\":[";
      for (int i = 0; i < 8; ++i) {
        char buf[64];
        std::snprintf(buf, sizeof buf, "%.17g", r2.next_unit());
        std::cout << (i ? "," : "") << buf;
      }
      da::Rng r3(7);
      da::Rng c = r3.fork();
      std::cout << "],\"fork7_child_u64\":\"" << c.next_u64() << "\",\"fork7_parent_next\":\""
                << r3.next_u64() << "\"}\n";
      return 0;
    }
    if (mode == "run") {
      if (argc < 9) throw da::ConfigError("run N P H D SEED SCHED OUTDIR [bf16] [exec]");
      const da::Index N = std::stol(argv[2]);
      const int P = std::stoi(argv[3]);
      const int H = std::stoi(argv[4]);
      const da::Index D = std::stol(argv[5]);
      const uint64_t seed = std::stoull(argv[6]);
      const std::string sched = argv[7];
      const std::string out = argv[8];
      const bool bf16 = argc > 9 && std::string(argv[9]) == "1";
      // exec: stepper (default) | concurrent | both (run both executors and
      // record whether every output is bit-identical, runtime.hpp:7-9)
      const std::string exec = argc > 10 ? argv[10] : "stepper";
      da::Rng rng(seed);
      std::vector<std::vector<double>> buf(9);
      std::ofstream meta(out + "/meta.json");
      meta << "{\"N\":" << N << ",\"P\":" << P << ",\"H\":" << H << ",\"D\":" << D
           << ",\"seed\":" << seed << ",\"schedule\":\"" << sched << "\",\"bf16\":" << bf16
           << ",\"heads\":[";
      for (int h = 0; h < H; ++h) {
        auto shards = make_head(P, N, D, rng, bf16);
        auto twin = shards;
        da::RunOptions opts;
        if (exec == "concurrent") opts.mode = da::ExecutorMode::Concurrent;
        const auto fr = da::run_forward(shards, pick(sched, P), opts);
        const auto bt = da::run_backward(shards, da::BackwardMode::Vanilla, opts);
        bool same = true;
        if (exec == "both") {
          da::RunOptions copts;
          copts.mode = da::ExecutorMode::Concurrent;
          copts.overlap = true;
          da::run_forward(twin, pick(sched, P), copts);
          da::run_backward(twin, da::BackwardMode::Vanilla, copts);
          auto eq = [](const auto& a, const auto& b) {
            if (a.size() != b.size()) return false;
            for (da::Index i = 0; i < a.size(); ++i)
              if (a.data()[i] != b.data()[i]) return false;
            return true;
          };
          for (int p = 0; p < P; ++p)
            same = same && eq(shards[p].out, twin[p].out) && eq(shards[p].lse, twin[p].lse) &&
                   eq(shards[p].dq, twin[p].dq) && eq(shards[p].dk, twin[p].dk) &&
                   eq(shards[p].dv, twin[p].dv);
        }
        for (const auto& s : shards) {
          const da::Matd* m[8] = {&s.q, &s.k, &s.v, &s.d_out, &s.out, &s.dq, &s.dk, &s.dv};
          const int slot[8] = {0, 1, 2, 3, 4, 6, 7, 8};
          for (int i = 0; i < 8; ++i)
            for (da::Index r = 0; r < m[i]->rows(); ++r)
              for (da::Index c = 0; c < m[i]->cols(); ++c) buf[slot[i]].push_back((*m[i])(r, c));
          for (da::Index r = 0; r < s.lse.size(); ++r) buf[5].push_back(s.lse(r));
        }
        const auto& fc = fr.trace.counters;
        const auto& bc = bt.counters;
        meta << (h ? "," : "") << "{\"fwd_counters\":[" << fc.kv_scalars << "," << fc.q_scalars
             << "," << fc.partial_scalars << "," << fc.grad_scalars << "," << fc.kv_messages
             << "," << fc.q_messages << "," << fc.partial_messages << "," << fc.grad_messages
             << "],\"bwd_counters\":[" << bc.kv_scalars << "," << bc.q_scalars << ","
             << bc.partial_scalars << "," << bc.grad_scalars << "," << bc.kv_messages << ","
             << bc.q_messages << "," << bc.partial_messages << "," << bc.grad_messages
             << "],\"fwd_kernel_calls\":" << fr.trace.attention_kernel_calls
             << ",\"bwd_kernel_calls\":" << bt.attention_kernel_calls
             << ",\"fwd_max_held\":" << fr.trace.max_remote_chunks_held
             << ",\"bwd_max_held\":" << bt.max_remote_chunks_held
             << ",\"fwd_makespan\":" << fr.trace.makespan << ",\"bwd_makespan\":"
             << bt.makespan << ",\"executors_bitwise_equal\":" << (same ? "true" : "false")
             << "}";
      }
      meta << "]}\n";
      const char* names[9] = {"q", "k", "v", "d_out", "out", "lse", "dq", "dk", "dv"};
      for (int i = 0; i < 9; ++i) write_bin(out + "/" + names[i] + ".bin", buf[i]);
      return 0;
    }
    if (mode == "time") {
      if (argc < 8) throw da::ConfigError("time N P H D SCHED THREADS");
      const da::Index N = std::stol(argv[2]);
      const int P = std::stoi(argv[3]);
      const int H = std::stoi(argv[4]);
      const da::Index D = std::stol(argv[5]);
      const std::string sched = argv[6];
      const int threads = std::max(1, std::stoi(argv[7]));
      da::Rng rng(0);
      std::vector<std::vector<da::SequenceShard>> heads;
      for (int h = 0; h < H; ++h) heads.push_back(make_head(P, N, D, rng, true));
      const int par = std::max(1, threads / P);  // heads in flight (P threads each)
      const auto t0 = std::chrono::steady_clock::now();
      std::vector<std::thread> pool;
      std::vector<std::exception_ptr> errs(H);
      for (int base = 0; base < H; base += par) {
        pool.clear();
        for (int h = base; h < std::min(H, base + par); ++h)
          pool.emplace_back([&, h] {
            try {
              da::RunOptions opts;
              opts.mode = da::ExecutorMode::Concurrent;
              da::run_forward(heads[h], pick(sched, P), opts);
              da::run_backward(heads[h], da::BackwardMode::Vanilla, opts);
            } catch (...) {
              errs[h] = std::current_exception();
            }
          });
        for (auto& t : pool) t.join();
      }
      for (auto& e : errs)
        if (e) std::rethrow_exception(e);
      const double secs =
          std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      const double flops = 7.0 * static_cast<double>(N) * N * D * H;
      std::printf("{\"seconds\":%.6f,\"flops\":%.6e,\"tflops\":%.6e,\"threads\":%d}\n", secs,
                  flops, flops / secs / 1e12, std::min(H, par) * P);  // threads actually running
      return 0;
    }
    std::cerr << "unknown mode " << mode << "\n";
    return 2;
  } catch (const da::ConfigError& e) {
    std::cerr << "config error: " << e.what() << "\n";
    return 2;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 1;
  }
}
