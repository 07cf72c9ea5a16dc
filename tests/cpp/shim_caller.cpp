// A C++ caller of the drop-in shim (include/xcls_gpu.hpp), written the way a user of the
// reference's xcls:: API writes it: `namespace xcls = xcls_gpu;` and the reference's types and
// free functions.  tests/test_gpu_cpp_shim.py compiles it with g++, links libxcls_gpu.so +
// libxknn.so, runs it on inputs it wrote to <dir>, and compares the outputs with the oracle.
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <string>
#include <vector>

#include "xcls_gpu.hpp"

namespace xcls = xcls_gpu;

template <typename T>
static std::vector<T> read_vec(const std::string& path) {
  std::ifstream f(path, std::ios::binary);
  f.seekg(0, std::ios::end);
  const std::size_t bytes = f.tellg();
  f.seekg(0);
  std::vector<T> v(bytes / sizeof(T));
  f.read(reinterpret_cast<char*>(v.data()), bytes);
  return v;
}
template <typename T>
static void write_vec(const std::string& path, const T* p, std::size_t n) {
  std::ofstream f(path, std::ios::binary);
  f.write(reinterpret_cast<const char*>(p), n * sizeof(T));
}

int main(int argc, char** argv) {
  if (argc < 2) return 2;
  const std::string dir = argv[1];
  const auto meta = read_vec<std::uint64_t>(dir + "/meta.bin");  // n, k, b, d, m, seed, shards
  const std::size_t n = meta[0], k = meta[1], b = meta[2], d = meta[3], m = meta[4], P = meta[6];
  const std::uint64_t seed = meta[5];
  xcls::KnnGraph g;
  g.num_classes = n;
  g.k = k;
  g.flat = read_vec<std::uint32_t>(dir + "/graph.bin");
  const auto labels = read_vec<std::uint32_t>(dir + "/labels.bin");
  const xcls::SelectionConfig cfg{m, seed};

  // select_active_classes over the full graph and over P compressed shards
  const xcls::ActiveSet full = xcls::select_active_classes(g, labels, cfg, n);
  write_vec(dir + "/sel_full.bin", full.class_indices.data(), full.size());
  std::vector<xcls::CompressedKnnGraph> shards;
  const xcls::ShardLayout layout{n, P};
  for (std::size_t s = 0; s < P; ++s) shards.push_back(xcls::compress_graph(g, layout, s));
  const xcls::ActiveSet act = xcls::select_active_classes(shards, labels, cfg, n);
  write_vec(dir + "/sel_span.bin", act.class_indices.data(), act.size());

  // knn_softmax_forward_backward on normalized inputs over that active set
  xcls::DenseMatrix x(b, d), w(n, d);
  x.data = read_vec<float>(dir + "/xnorm.bin");
  w.data = read_vec<float>(dir + "/wnorm.bin");
  const xcls::LossAndGrad lg = xcls::knn_softmax_forward_backward(x, w, labels, act, 30.0f);
  write_vec(dir + "/fb_loss.bin", &lg.loss, 1);
  write_vec(dir + "/fb_gf.bin", lg.grad_features.data.data(), lg.grad_features.data.size());
  write_vec(dir + "/fb_gw.bin", lg.grad_weights.data.data(), lg.grad_weights.data.size());

  // the fc half of HybridSim with P simulated workers' graphs, fp32 tensor-core precision
  xcls::FcOptions opt;
  opt.selection = cfg;
  opt.max_batch = b;
  opt.precision = XKNN_PREC_FP32;
  xcls::HybridSimFc sim(n, d, opt);
  sim.set_shard_graphs(shards);
  xcls::DenseMatrix w0(n, d);
  w0.data = read_vec<float>(dir + "/wraw.bin");
  sim.load_model(w0);
  xcls::DenseMatrix f(b, d);
  f.data = read_vec<float>(dir + "/feat.bin");
  std::vector<double> losses;
  xcls::DenseMatrix gfeat;
  for (int step = 0; step < 2; ++step) losses.push_back(sim.train_step(f, labels, 0.1f, &gfeat).loss);
  write_vec(dir + "/sim_loss.bin", losses.data(), losses.size());
  const xcls::DenseMatrix wt = sim.fc_weights();
  write_vec(dir + "/sim_w.bin", wt.data.data(), wt.data.size());
  write_vec(dir + "/sim_gf.bin", gfeat.data.data(), gfeat.data.size());

  // the reference's error classes surface as the same exception types
  int errs = 0;
  try {
    xcls::select_active_classes(g, labels, xcls::SelectionConfig{1, seed}, n);
  } catch (const xcls::MTooSmall&) {
    errs |= 1;
  }
  try {
    std::vector<std::uint32_t> bad(labels);
    bad[0] = static_cast<std::uint32_t>(n);
    xcls::select_active_classes(shards, bad, cfg, n);
  } catch (const xcls::LabelOutOfRange&) {
    errs |= 2;
  }
  try {
    xcls::ActiveSet small;
    small.class_indices = {act.class_indices[0]};
    xcls::knn_softmax_forward_backward(x, w, labels, small, 30.0f);
  } catch (const xcls::LabelNotActive&) {
    errs |= 4;
  }
  write_vec(dir + "/errs.bin", &errs, 1);
  std::cout << "shim_caller ok, errs=" << errs << std::endl;
  return 0;
}
