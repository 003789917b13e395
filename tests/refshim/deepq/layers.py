from paper_1804_05834_b200.network import LayerSpec  # noqa: F401


def make_layer(spec, name):
    """deepq.layers.make_layer: the device Network takes (name, spec) pairs."""
    return (name, spec)
