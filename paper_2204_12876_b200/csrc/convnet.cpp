// Conv-net traversability model: validation and the weight-file reader
// (reference analysis.cpp:27-39 and 218-290). Grammar, per content line
// (blank lines and '#' comments skipped):
//   layers: <n>
//   then n times:  kernel: <k>  /  k rows of k numbers  /  bias: <b>  /
//                  activation: relu|sigmoid|identity
// Numbers go through the same libstdc++ conversions as the reference
// (std::stod for tagged values, operator>> for kernel rows), so a file is
// accepted or rejected identically, with the same messages.
#include <cmath>
#include <fstream>
#include <sstream>

#include "relief_internal.hpp"

namespace rb200 {

void ConvNetSpec::validate() const {
  if (layers.empty()) fail(Err::kInvalidModel, "model has no layers");
  for (const ConvLayer& l : layers) {
    if (l.kernel_size < 1 || l.kernel_size % 2 == 0)
      fail(Err::kInvalidModel, "kernel size must be odd and positive");
    if (l.kernel.size() != static_cast<std::size_t>(l.kernel_size) * l.kernel_size)
      fail(Err::kInvalidModel, "kernel element count mismatch");
    for (const double w : l.kernel)
      if (!std::isfinite(w)) fail(Err::kInvalidModel, "non-finite kernel weight");
    if (!std::isfinite(l.bias)) fail(Err::kInvalidModel, "non-finite bias");
  }
}

namespace {

// static_cast<int>(double) as x86-64 executes it (cvttsd2si: out of range and
// NaN give INT_MIN), which is what the reference binary does for absurd counts.
int toIntX86(double v) {
  if (!(v >= -2147483648.0 && v < 2147483648.0)) return INT32_MIN;
  return static_cast<int>(v);
}

class ModelReader {
 public:
  explicit ModelReader(std::istream& in) : in_(in) {}

  // Next line that is neither blank nor a comment, from its first non-blank.
  std::string content() {
    std::string line;
    while (std::getline(in_, line)) {
      ++line_no_;
      const std::size_t first = line.find_first_not_of(" \t\r");
      if (first == std::string::npos || line[first] == '#') continue;
      return line.substr(first);
    }
    fail(Err::kInvalidModel, "unexpected end of model file at line " + std::to_string(line_no_));
  }

  // The reference passes line_no by value next to nextContentLine(in,
  // line_no) in one call (analysis.cpp:236-237,242-243,258); g++ evaluates
  // that argument first, so tag / number errors name the line number as it
  // was BEFORE the tagged line was read. Reproduced for identical messages.
  double tagged(const std::string& tag) {
    const int reported = line_no_;
    const std::string line = content();
    if (line.compare(0, tag.size(), tag) != 0)
      fail(Err::kInvalidModel, "expected '" + tag + "' at line " + std::to_string(reported));
    try {
      return std::stod(line.substr(tag.size()));
    } catch (const std::exception&) {
      fail(Err::kInvalidModel, "bad number at line " + std::to_string(reported));
    }
  }

  void row(int k, std::vector<double>& out) {
    std::istringstream fields(content());
    for (int c = 0; c < k; ++c) {
      double v;
      if (!(fields >> v))
        fail(Err::kInvalidModel, "kernel row too short at line " + std::to_string(line_no_));
      out.push_back(v);
    }
  }

  Activation activation() {
    static const std::string tag = "activation:";
    const std::string line = content();
    if (line.compare(0, tag.size(), tag) != 0)
      fail(Err::kInvalidModel, "expected 'activation:' at line " + std::to_string(line_no_));
    std::string name = line.substr(tag.size());
    name.erase(0, name.find_first_not_of(" \t"));
    name.erase(name.find_last_not_of(" \t\r") + 1);
    if (name == "relu") return Activation::kRelu;
    if (name == "sigmoid") return Activation::kSigmoid;
    if (name == "identity") return Activation::kIdentity;
    fail(Err::kInvalidModel,
         "unknown activation '" + name + "' at line " + std::to_string(line_no_));
  }

  int line() const { return line_no_; }

 private:
  std::istream& in_;
  int line_no_ = 0;
};

ConvNetSpec readModel(std::istream& in) {
  ModelReader rd(in);
  ConvNetSpec spec;
  const int n_layers = toIntX86(rd.tagged("layers:"));
  if (n_layers < 1) fail(Err::kInvalidModel, "layer count must be >= 1");
  for (int li = 0; li < n_layers; ++li) {
    ConvLayer layer;
    layer.kernel_size = toIntX86(rd.tagged("kernel:"));
    if (layer.kernel_size < 1 || layer.kernel_size % 2 == 0)
      fail(Err::kInvalidModel, "kernel size must be odd, line " + std::to_string(rd.line()));
    for (int r = 0; r < layer.kernel_size; ++r) rd.row(layer.kernel_size, layer.kernel);
    layer.bias = rd.tagged("bias:");
    layer.activation = rd.activation();
    spec.layers.push_back(std::move(layer));
  }
  spec.validate();
  return spec;
}

}  // namespace

ConvNetSpec loadConvNetSpecText(const std::string& text) {
  std::istringstream in(text);
  return readModel(in);
}

ConvNetSpec loadConvNetSpecFile(const std::string& path) {
  std::ifstream in(path);
  if (!in) fail(Err::kIo, "cannot open model file: " + path);
  return readModel(in);
}

}  // namespace rb200
